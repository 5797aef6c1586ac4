// Multicast (NVLS) diagnosis through the driver API from C.
// Round 1 only probed through cuda-python; this walks every parameter the
// driver checks (handle type, numDevices, size vs granularity, flags) and, if
// an object can be created, runs the whole NVLS data path on one device:
// cuMulticastAddDevice -> cuMemCreate -> cuMulticastBindMem -> cuMemMap of the
// multicast handle -> multimem.ld_reduce / multimem.st from a kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/probe_mc scripts/probe_multicast.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

static const char* ename(CUresult r) {
    const char* s = nullptr;
    cuGetErrorName(r, &s);
    return s ? s : "?";
}
#define CK(x) do { CUresult _r = (x); if (_r != CUDA_SUCCESS) { printf("  %-40s -> %s (%d)\n", #x, ename(_r), (int)_r); return _r; } } while (0)

__global__ void mm_reduce(float* mc, float* uc, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i * 4 >= n) return;
    float4 v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(mc + 4 * i) : "memory");
    v.x += 1.f; v.y += 1.f; v.z += 1.f; v.w += 1.f;
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(mc + 4 * i), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
    (void)uc;
}

static CUresult full_path(CUdevice dev, CUmemAllocationHandleType ht, int ndev) {
    CUmulticastObjectProp mp;
    memset(&mp, 0, sizeof(mp));
    mp.numDevices = ndev;
    mp.handleTypes = ht;
    size_t g = 0;
    CK(cuMulticastGetGranularity(&g, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    mp.size = g;
    CUmemGenericAllocationHandle mc;
    CK(cuMulticastCreate(&mc, &mp));
    printf("  create OK (size %zu)\n", g);
    CK(cuMulticastAddDevice(mc, dev));
    printf("  add device OK\n");
    CUmemAllocationProp ap;
    memset(&ap, 0, sizeof(ap));
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = (int)dev;
    ap.requestedHandleTypes = ht;
    size_t ag = 0;
    CK(cuMemGetAllocationGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    CUmemGenericAllocationHandle ph;
    CK(cuMemCreate(&ph, g, &ap, 0));
    CK(cuMulticastBindMem(mc, 0, ph, 0, g, 0));
    printf("  bind OK\n");
    CUdeviceptr uva = 0, mva = 0;
    CK(cuMemAddressReserve(&uva, g, g, 0, 0));
    CK(cuMemMap(uva, g, 0, ph, 0));
    CK(cuMemAddressReserve(&mva, g, g, 0, 0));
    CK(cuMemMap(mva, g, 0, mc, 0));
    CUmemAccessDesc acc;
    memset(&acc, 0, sizeof(acc));
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = (int)dev;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(uva, g, &acc, 1));
    CK(cuMemSetAccess(mva, g, &acc, 1));
    int n = 1 << 16;
    float h[16];
    for (int i = 0; i < 16; ++i) h[i] = (float)i;
    cudaMemset((void*)uva, 0, n * 4);
    cudaMemcpy((void*)uva, h, sizeof(h), cudaMemcpyHostToDevice);
    mm_reduce<<<n / 4 / 256, 256>>>((float*)mva, (float*)uva, n);
    cudaError_t e = cudaDeviceSynchronize();
    printf("  multimem kernel: %s\n", cudaGetErrorString(e));
    cudaMemcpy(h, (void*)uva, sizeof(h), cudaMemcpyDeviceToHost);
    printf("  uc[0..3] after ld_reduce+1 / st: %g %g %g %g (expect 1 2 3 4)\n", h[0], h[1], h[2], h[3]);
    return CUDA_SUCCESS;
}

int main() {
    CUresult r = cuInit(0);
    printf("cuInit %s\n", ename(r));
    int drv = 0;
    cuDriverGetVersion(&drv);
    printf("driver API version %d\n", drv);
    CUdevice dev;
    cuDeviceGet(&dev, 0);
    char name[128];
    cuDeviceGetName(name, sizeof(name), dev);
    printf("device 0: %s\n", name);
    struct { const char* n; CUdevice_attribute a; } attrs[] = {
        {"MULTICAST_SUPPORTED", CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED},
        {"HANDLE_TYPE_FABRIC_SUPPORTED", CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED},
        {"HANDLE_TYPE_POSIX_FD_SUPPORTED", CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED},
        {"VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED", CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED},
    };
    for (auto& a : attrs) {
        int v = -1;
        CUresult e = cuDeviceGetAttribute(&v, a.a, dev);
        printf("attr %-36s = %d (%s)\n", a.n, v, ename(e));
    }
    CUcontext ctx;
    cuDevicePrimaryCtxRetain(&ctx, dev);
    cuCtxSetCurrent(ctx);
    cudaSetDevice(0);
    struct { const char* n; CUmemAllocationHandleType h; } hts[] = {
        {"NONE", CU_MEM_HANDLE_TYPE_NONE},
        {"POSIX_FD", CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR},
        {"FABRIC", CU_MEM_HANDLE_TYPE_FABRIC},
    };
    for (auto& h : hts) {
        for (int nd = 1; nd <= 2; ++nd) {
            for (int sz_mult = 1; sz_mult <= 16; sz_mult *= 16) {
                CUmulticastObjectProp mp;
                memset(&mp, 0, sizeof(mp));
                mp.numDevices = nd;
                mp.handleTypes = h.h;
                size_t gmin = 0, grec = 0;
                CUresult e1 = cuMulticastGetGranularity(&gmin, &mp, CU_MULTICAST_GRANULARITY_MINIMUM);
                CUresult e2 = cuMulticastGetGranularity(&grec, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED);
                mp.size = grec * sz_mult;
                CUmemGenericAllocationHandle mc = 0;
                CUresult e3 = cuMulticastCreate(&mc, &mp);
                printf("create ht=%-8s numDevices=%d size=%zu (gran min %zu %s rec %zu %s) -> %s\n", h.n, nd, mp.size,
                       gmin, ename(e1), grec, ename(e2), ename(e3));
                if (e3 == CUDA_SUCCESS) cuMemRelease(mc);
            }
        }
    }
    for (auto& h : hts) {
        printf("full NVLS path, ht=%s numDevices=1:\n", h.n);
        full_path(dev, h.h, 1);
    }
    return 0;
}
