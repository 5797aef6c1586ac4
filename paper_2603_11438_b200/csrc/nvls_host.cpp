// NVLS host side: one multicast object per real comm,
// bound to a region of every rank's memory (nvls.cu runs the switch reduction).
//
//   rank 0   cuMulticastCreate(numDevices = nranks) and export: a FABRIC handle
//            (64 B, travels through the bootstrap all-gather) or, where fabric
//            handles are refused, a POSIX file descriptor that the peers copy
//            out of rank 0's process with pidfd_getfd(2);
//   all      import, cuMulticastAddDevice(own device)        (all-gather = barrier)
//   all      cuMemCreate + cuMulticastBindMem, map the physical memory (unicast)
//            and the multicast object (multicast) into this process
//
// Every rank runs the same number of all-gathers whatever fails locally, so a
// failure anywhere leaves every rank without NVLS (and the comm itself works):
// the first failing call, its CUresult name and the rank are kept in `why`
// (polar_comm_nvls_info).  Driver entry points come through the runtime, so
// libpolar does not link libcuda.
#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <vector>

#include "polar.h"
#include "polar_internal.h"

#ifndef SYS_pidfd_open
#define SYS_pidfd_open 434
#endif
#ifndef SYS_pidfd_getfd
#define SYS_pidfd_getfd 438
#endif

namespace polar {

namespace {

std::atomic<int> g_nvls_comms{0};

template <class F> F drv(const char* name) {
    cudaDriverEntryPointQueryResult q;
    void* fp = nullptr;
    if (cudaGetDriverEntryPoint(name, &fp, cudaEnableDefault, &q) != cudaSuccess || !fp) return nullptr;
    return reinterpret_cast<F>(fp);
}

struct Drv {
    CUresult (*getErrorName)(CUresult, const char**) = nullptr;
    CUresult (*devAttr)(int*, CUdevice_attribute, CUdevice) = nullptr;
    CUresult (*mcGran)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
    CUresult (*mcCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
    CUresult (*mcAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
    CUresult (*mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                          unsigned long long) = nullptr;
    CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
    CUresult (*memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
    CUresult (*memRelease)(CUmemGenericAllocationHandle) = nullptr;
    CUresult (*memExport)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long) = nullptr;
    CUresult (*memImport)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
    CUresult (*addrReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
    CUresult (*addrFree)(CUdeviceptr, size_t) = nullptr;
    CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
    CUresult (*memUnmap)(CUdeviceptr, size_t) = nullptr;
    CUresult (*memSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
    bool ok = false;
    Drv() {
        getErrorName = drv<decltype(getErrorName)>("cuGetErrorName");
        devAttr = drv<decltype(devAttr)>("cuDeviceGetAttribute");
        mcGran = drv<decltype(mcGran)>("cuMulticastGetGranularity");
        mcCreate = drv<decltype(mcCreate)>("cuMulticastCreate");
        mcAddDevice = drv<decltype(mcAddDevice)>("cuMulticastAddDevice");
        mcBindMem = drv<decltype(mcBindMem)>("cuMulticastBindMem");
        mcUnbind = drv<decltype(mcUnbind)>("cuMulticastUnbind");
        memCreate = drv<decltype(memCreate)>("cuMemCreate");
        memRelease = drv<decltype(memRelease)>("cuMemRelease");
        memExport = drv<decltype(memExport)>("cuMemExportToShareableHandle");
        memImport = drv<decltype(memImport)>("cuMemImportFromShareableHandle");
        addrReserve = drv<decltype(addrReserve)>("cuMemAddressReserve");
        addrFree = drv<decltype(addrFree)>("cuMemAddressFree");
        memMap = drv<decltype(memMap)>("cuMemMap");
        memUnmap = drv<decltype(memUnmap)>("cuMemUnmap");
        memSetAccess = drv<decltype(memSetAccess)>("cuMemSetAccess");
        ok = getErrorName && devAttr && mcGran && mcCreate && mcAddDevice && mcBindMem && mcUnbind && memCreate &&
             memRelease && memExport && memImport && addrReserve && addrFree && memMap && memUnmap && memSetAccess;
    }
    const char* name(CUresult r) const {
        const char* s = nullptr;
        if (getErrorName) getErrorName(r, &s);
        return s ? s : "CUDA_ERROR_?";
    }
};

const Drv& D() {
    static Drv d;
    return d;
}

// one all-gather record per step
struct Msg {
    int32_t ok;          // 1: this rank's step succeeded
    int32_t result;      // CUresult of the failing call
    int32_t htype;       // rank 0, step B: CU_MEM_HANDLE_TYPE_FABRIC or _POSIX_FILE_DESCRIPTOR
    int32_t fd;          // rank 0, step B: its file descriptor (POSIX)
    int32_t pid;         // rank 0, step B: its pid (POSIX)
    int32_t pad;
    uint64_t size;       // rank 0, step B: bound bytes per rank
    char what[40];       // the failing call
    unsigned char fabric[64];
};
static_assert(sizeof(Msg) == 136, "nvls bootstrap record");

bool gather(polar_allgather_fn ag, void* user, int nranks, const Msg& mine, std::vector<Msg>& all) {
    all.assign(nranks, Msg{});
    return ag(&mine, all.data(), sizeof(Msg), user) == 0;
}

// first failing rank of a step -> s.why
bool all_ok(NvlsState& s, const std::vector<Msg>& all, const char* step) {
    for (size_t p = 0; p < all.size(); ++p)
        if (!all[p].ok) {
            std::snprintf(s.why, sizeof(s.why), "%s: %s -> %s (rank %zu)", step, all[p].what,
                          D().name((CUresult)all[p].result), p);
            s.status = all[p].result ? all[p].result : -1;
            return false;
        }
    return true;
}

void fail(Msg& m, const char* what, CUresult r) {
    m.ok = 0;
    m.result = (int32_t)r;
    std::snprintf(m.what, sizeof(m.what), "%s", what);
}

void release_local(NvlsState& s, int device) {
    const Drv& d = D();
    if (!d.ok) return;
    if (s.mc) { d.memUnmap((CUdeviceptr)s.mc, s.bytes); d.addrFree((CUdeviceptr)s.mc, s.bytes); }
    if (s.uc) { d.memUnmap((CUdeviceptr)s.uc, s.bytes); d.addrFree((CUdeviceptr)s.uc, s.bytes); }
    if (s.bound) d.mcUnbind((CUmemGenericAllocationHandle)s.mc_handle, (CUdevice)device, 0, s.bytes);
    if (s.phys) d.memRelease((CUmemGenericAllocationHandle)s.phys);
    if (s.mc_handle) d.memRelease((CUmemGenericAllocationHandle)s.mc_handle);
    if (s.fd >= 0) close(s.fd);
    s.mc = s.uc = nullptr;
    s.phys = s.mc_handle = 0;
    s.bound = false;
    s.fd = -1;
}

}  // namespace

polar_status nvls_setup(NvlsState& s, int nranks, int rank, int device, polar_allgather_fn ag, void* user,
                        size_t want_bytes) {
    s = NvlsState{};
    const Drv& d = D();
    std::vector<Msg> all;
    // ---- A: every device supports multicast (and the driver entry points exist)
    Msg a{};
    a.ok = 1;
    if (!d.ok) {
        fail(a, "driver entry points", CUDA_ERROR_NOT_SUPPORTED);
    } else {
        int v = 0;
        CUresult r = d.devAttr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, (CUdevice)device);
        if (r != CUDA_SUCCESS || !v) fail(a, "CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", r ? r : CUDA_ERROR_NOT_SUPPORTED);
    }
    if (!gather(ag, user, nranks, a, all)) return POLAR_ESTATE;
    if (!all_ok(s, all, "support")) return POLAR_OK;
    // ---- B: rank 0 creates the object and exports a shareable handle
    Msg b{};
    b.ok = 1;
    b.fd = -1;
    CUmulticastObjectProp mp;
    std::memset(&mp, 0, sizeof(mp));
    mp.numDevices = (unsigned)nranks;
    CUmemGenericAllocationHandle mc = 0;
    if (rank == 0) {
        static const CUmemAllocationHandleType kTypes[2] = {CU_MEM_HANDLE_TYPE_FABRIC,
                                                             CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR};
        CUresult r = CUDA_ERROR_UNKNOWN;
        const char* what = "cuMulticastCreate";
        for (CUmemAllocationHandleType ht : kTypes) {
            mp.handleTypes = ht;
            size_t g = 0;
            r = d.mcGran(&g, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED);
            if (r != CUDA_SUCCESS) { what = "cuMulticastGetGranularity"; continue; }
            mp.size = (want_bytes + g - 1) / g * g;
            r = d.mcCreate(&mc, &mp);
            if (r != CUDA_SUCCESS) { what = "cuMulticastCreate"; mc = 0; continue; }
            if (ht == CU_MEM_HANDLE_TYPE_FABRIC) {
                CUmemFabricHandle fh;
                r = d.memExport(&fh, mc, ht, 0);
                if (r == CUDA_SUCCESS) std::memcpy(b.fabric, &fh, sizeof(b.fabric));
            } else {
                int fd = -1;
                r = d.memExport(&fd, mc, ht, 0);
                b.fd = fd;
                b.pid = (int32_t)getpid();
            }
            if (r != CUDA_SUCCESS) { what = "cuMemExportToShareableHandle"; d.memRelease(mc); mc = 0; continue; }
            b.htype = (int32_t)ht;
            b.size = mp.size;
            break;
        }
        if (!mc) fail(b, what, r);
    }
    if (!gather(ag, user, nranks, b, all)) { if (mc) d.memRelease(mc); return POLAR_ESTATE; }
    if (!all_ok(s, all, "create")) return POLAR_OK;
    const Msg& r0 = all[0];
    s.bytes = (size_t)r0.size;
    s.handle_type = r0.htype;
    // ---- C: import (peers) and add this rank's device
    Msg c{};
    c.ok = 1;
    if (rank == 0) {
        s.mc_handle = (unsigned long long)mc;
        s.fd = r0.fd;
    } else if (r0.htype == CU_MEM_HANDLE_TYPE_FABRIC) {
        CUmemFabricHandle fh;
        std::memcpy(&fh, r0.fabric, sizeof(r0.fabric));
        CUmemGenericAllocationHandle h = 0;
        CUresult r = d.memImport(&h, &fh, CU_MEM_HANDLE_TYPE_FABRIC);
        if (r != CUDA_SUCCESS) fail(c, "cuMemImportFromShareableHandle", r);
        s.mc_handle = (unsigned long long)h;
    } else {
        const int pidfd = (int)syscall(SYS_pidfd_open, (pid_t)r0.pid, 0);
        const int fd = pidfd >= 0 ? (int)syscall(SYS_pidfd_getfd, pidfd, r0.fd, 0) : -1;
        if (pidfd >= 0) close(pidfd);
        if (fd < 0) {
            fail(c, "pidfd_getfd", CUDA_ERROR_NOT_PERMITTED);
        } else {
            CUmemGenericAllocationHandle h = 0;
            CUresult r = d.memImport(&h, reinterpret_cast<void*>((uintptr_t)fd), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
            close(fd);
            if (r != CUDA_SUCCESS) fail(c, "cuMemImportFromShareableHandle", r);
            s.mc_handle = (unsigned long long)h;
        }
    }
    if (c.ok) {
        CUresult r = d.mcAddDevice((CUmemGenericAllocationHandle)s.mc_handle, (CUdevice)device);
        if (r != CUDA_SUCCESS) fail(c, "cuMulticastAddDevice", r);
    }
    if (!gather(ag, user, nranks, c, all)) { release_local(s, device); return POLAR_ESTATE; }
    if (!all_ok(s, all, "join")) { release_local(s, device); return POLAR_OK; }
    // ---- D: bind this rank's physical memory, map it and the multicast object
    Msg m{};
    m.ok = 1;
    {
        CUmemAllocationProp ap;
        std::memset(&ap, 0, sizeof(ap));
        ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ap.location.id = device;
        CUmemGenericAllocationHandle ph = 0;
        CUdeviceptr uva = 0, mva = 0;
        CUresult r = d.memCreate(&ph, s.bytes, &ap, 0);
        if (r != CUDA_SUCCESS) { fail(m, "cuMemCreate", r); goto done; }
        s.phys = (unsigned long long)ph;
        r = d.mcBindMem((CUmemGenericAllocationHandle)s.mc_handle, 0, ph, 0, s.bytes, 0);
        if (r != CUDA_SUCCESS) { fail(m, "cuMulticastBindMem", r); goto done; }
        s.bound = true;
        CUmemAccessDesc acc;
        std::memset(&acc, 0, sizeof(acc));
        acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        acc.location.id = device;
        acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        r = d.addrReserve(&uva, s.bytes, 0, 0, 0);   // default alignment (the size need not be a power of two)
        if (r != CUDA_SUCCESS) { fail(m, "cuMemAddressReserve", r); goto done; }
        r = d.memMap(uva, s.bytes, 0, ph, 0);
        if (r != CUDA_SUCCESS) { d.addrFree(uva, s.bytes); fail(m, "cuMemMap(unicast)", r); goto done; }
        s.uc = reinterpret_cast<char*>(uva);
        r = d.memSetAccess(uva, s.bytes, &acc, 1);
        if (r != CUDA_SUCCESS) { fail(m, "cuMemSetAccess(unicast)", r); goto done; }
        r = d.addrReserve(&mva, s.bytes, 0, 0, 0);
        if (r != CUDA_SUCCESS) { fail(m, "cuMemAddressReserve", r); goto done; }
        r = d.memMap(mva, s.bytes, 0, (CUmemGenericAllocationHandle)s.mc_handle, 0);
        if (r != CUDA_SUCCESS) { d.addrFree(mva, s.bytes); fail(m, "cuMemMap(multicast)", r); goto done; }
        s.mc = reinterpret_cast<char*>(mva);
        r = d.memSetAccess(mva, s.bytes, &acc, 1);
        if (r != CUDA_SUCCESS) { fail(m, "cuMemSetAccess(multicast)", r); goto done; }
        if (cudaMemset(s.uc, 0, s.bytes) != cudaSuccess) { fail(m, "cudaMemset", CUDA_ERROR_UNKNOWN); goto done; }
    }
done:
    if (!gather(ag, user, nranks, m, all)) { release_local(s, device); return POLAR_ESTATE; }
    if (!all_ok(s, all, "bind")) { release_local(s, device); return POLAR_OK; }
    s.ok = true;
    std::snprintf(s.why, sizeof(s.why), "multicast object over %d GPUs, %zu bytes bound per rank (%s handle)", nranks,
                  s.bytes, s.handle_type == CU_MEM_HANDLE_TYPE_FABRIC ? "fabric" : "posix-fd");
    g_nvls_comms.fetch_add(1);
    return POLAR_OK;
}

void nvls_teardown(NvlsState& s, int device) {
    if (s.ok) g_nvls_comms.fetch_sub(1);
    release_local(s, device);
    s.ok = false;
}

bool nvls_available() { return g_nvls_comms.load() > 0; }

}  // namespace polar

extern "C" int polar_nvls_available(void) { return polar::nvls_available() ? 1 : 0; }
