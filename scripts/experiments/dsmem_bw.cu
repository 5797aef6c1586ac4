// Microbenchmark: distributed-shared-memory push bandwidth per SM on B200
// (clusters of 8 CTAs, one per SM; CTA r pushes to CTA r+1 of its cluster).
//   mode 0: st.async.v4 from registers, complete_tx on the receiver's mbarrier
//   mode 1: st.shared::cluster.v4 (plain remote stores), cluster barrier at the end
//   mode 2: cp.async.bulk.shared::cluster.shared::cta (one thread, 16 KiB chunks)
//   mode 3: ld.shared::cluster.v4 pull from the predecessor (reads)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_bw dsmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kCl = 8;
constexpr unsigned kBuf = 64 << 10;        // receive region per CTA
constexpr unsigned kPhase = 1u << 19;      // bytes per mbarrier phase (< 2^20 tx limit)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
    uint32_t o;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
    return o;
}
__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t par) {
    uint32_t ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}"
                 : "=r"(ok) : "r"(bar), "r"(par) : "memory");
    return ok;
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) push(unsigned long long bytes_per_cta, unsigned long long* cycles) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const uint32_t succ = (rank + 1) % kCl, pred = (rank + kCl - 1) % kCl;
    const uint32_t buf = smem_u32(sm), b = smem_u32(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    for (unsigned i = threadIdx.x; i < kBuf / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i;
    csync();
    const uint32_t rbuf = mapa(buf, succ), rbar = mapa(b, succ), pbuf = mapa(buf, pred);
    const unsigned long long t0 = clock64();
    const unsigned nph = (unsigned)(bytes_per_cta / kPhase);
    uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    uint32_t acc = 0;
    for (unsigned ph = 0; ph < nph; ++ph) {
        if (MODE == 0 || MODE == 2) {
            if (threadIdx.x == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kPhase));
        }
        if (MODE == 0) {
            for (unsigned o = threadIdx.x * 16; o < kPhase; o += blockDim.x * 16)
                asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%2,%3,%4}, [%5];" ::"r"(
                                 rbuf + (o % kBuf)),
                             "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rbar)
                             : "memory");
        } else if (MODE == 1) {
            for (unsigned o = threadIdx.x * 16; o < kPhase; o += blockDim.x * 16)
                asm volatile("st.shared::cluster.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(rbuf + (o % kBuf)), "r"(v.x), "r"(v.y),
                             "r"(v.z), "r"(v.w)
                             : "memory");
        } else if (MODE == 2) {
            if (threadIdx.x == 0)
                for (unsigned o = 0; o < kPhase; o += 16384)
                    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                     rbuf + (o % kBuf)),
                                 "r"(buf + ((o + 16384) % kBuf)), "r"(16384u), "r"(rbar)
                                 : "memory");
        } else {
            for (unsigned o = threadIdx.x * 16; o < kPhase; o += blockDim.x * 16) {
                uint4 w;
                asm volatile("ld.shared::cluster.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                             : "r"(pbuf + (o % kBuf)) : "memory");
                acc += w.x ^ w.w;
            }
        }
        if (MODE == 0 || MODE == 2) {
            while (!try_wait(b, ph & 1)) {}
        }
    }
    csync();
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0 + (acc == 0xdeadbeef);
}

int main(int argc, char** argv) {
    const int nclusters = argc > 1 ? atoi(argv[1]) : 15;
    const unsigned long long bytes = 64ull << 20;   // per CTA
    unsigned long long* d;
    cudaMalloc(&d, sizeof(unsigned long long) * 8 * 64);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    void (*fns[4])(unsigned long long, unsigned long long*) = {push<0>, push<1>, push<2>, push<3>};
    const char* names[4] = {"st.async", "st.shared::cluster", "cp.async.bulk", "ld.shared::cluster"};
    const int m0 = argc > 2 ? atoi(argv[2]) : 0, m1 = argc > 2 ? m0 + 1 : 4;
    for (int m = m0; m < m1; ++m) {
        cudaFuncSetAttribute(fns[m], cudaFuncAttributeMaxDynamicSharedMemorySize, kBuf);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(nclusters * kCl);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = kBuf;
        cudaLaunchAttribute a{};
        a.id = cudaLaunchAttributeClusterDimension;
        a.val.clusterDim.x = kCl; a.val.clusterDim.y = 1; a.val.clusterDim.z = 1;
        cfg.attrs = &a;
        cfg.numAttrs = 1;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            cudaError_t err = cudaLaunchKernelEx(&cfg, fns[m], bytes, d);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            cudaError_t e2 = cudaGetLastError();
            if (err != cudaSuccess || e2 != cudaSuccess) { printf("%s: error %s / %s\n", names[m], cudaGetErrorString(err), cudaGetErrorString(e2)); break; }
            if (rep == 1)
                printf("{\"mode\": \"%s\", \"clusters\": %d, \"ms\": %.3f, \"per_sm_gbs\": %.1f, \"per_sm_B_per_clk\": %.1f, \"total_gbs\": %.0f}\n",
                       names[m], nclusters, ms, bytes / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / (clk * 1e3),
                       bytes * nclusters * kCl / (ms * 1e-3) / 1e9);
        }
    }
    return 0;
}
