// Communicators, symmetric memory, dispatch (include/polar.h).
//
// polar_allreduce: validate -> polar_decide (the tuner hook)
// -> pick the kernel instance <dtype, op, algo, proto> -> ONE launch of
// nlocal x nchannels CTAs on the caller's stream.  No host sync, no per-call
// allocation.  Real comms map every peer's scratch with CUDA IPC (the only
// host collective is the init/registration all-gather); virtual comms host all
// ranks on one device and use a cooperative launch.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "device.cuh"
#include "dispatch.h"
#include "p2p_probe.cuh"
#include "polar.h"
#include "polar_internal.h"

namespace polar {

namespace dev {
// init barrier: CTA b (local rank) signals every peer and waits for all
__global__ void init_barrier_kernel(Params P, unsigned long long value) {
    const int r = P.rank0 + (int)blockIdx.x;
    const int tid = (int)threadIdx.x;
    if (tid < P.nranks) st_release(flag_ptr(P, tid, F_INIT, 0, r), value, P.sys);
    bool ok = true;
    if (tid < P.nranks) ok = wait_geq(P, flag_ptr(P, r, F_INIT, 0, tid), value);
    __syncthreads_and(ok);
}
}  // namespace dev

const void* init_barrier_kernel_ptr() { return reinterpret_cast<const void*>(&dev::init_barrier_kernel); }

static size_t env_size(const char* name, size_t dflt) {
    const char* v = std::getenv(name);
    if (!v || !*v) return dflt;
    char* end = nullptr;
    unsigned long long x = std::strtoull(v, &end, 0);
    return x ? (size_t)x : dflt;
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

Layout make_layout(bool with_bounce) {
    Layout L{};
    size_t off = 0;
    L.flags_off = off; off = align_up(off + kFlagBytes, 4096);
    L.state_off = off; off = align_up(off + kStateBytes, 4096);
    L.tags_off = off; off = align_up(off + kTagRing * 16, 4096);
    L.os_chunk = align_up(env_size("POLAR_OS_CHUNK", 1 << 20), 512);
    L.os_off = off; off = align_up(off + 2 * kMaxRanks * L.os_chunk, 4096);
    L.osll_chunk = align_up(env_size("POLAR_OSLL_CHUNK", 256 << 10), 512);
    L.osll_off = off; off = align_up(off + 2 * kMaxRanks * 2 * L.osll_chunk, 4096);
    L.tsll_chunk = align_up(env_size("POLAR_TSLL_CHUNK", 256 << 10), 512);
    L.tsll_off = off; off = align_up(off + 2 * (2 * kMaxRanks * 2 * L.tsll_chunk), 4096);
    L.ring_slot = align_up(env_size("POLAR_RING_SLOT", 120 << 10), 512);   // 7680 f32 packs: whole 480-thread x 4-pack batches per half slot (ring_simple_ws)
    L.ring_off = off; off = align_up(off + (size_t)kMaxCh * kSteps * L.ring_slot, 4096);
    L.ringll_slot = align_up(env_size("POLAR_RINGLL_SLOT", 64 << 10), 512);
    L.ringll_off = off; off = align_up(off + (size_t)kMaxCh * kSteps * L.ringll_slot, 4096);
    L.tree_slot = align_up(env_size("POLAR_TREE_SLOT", 120 << 10), 512);   // whole 480-thread batches per half slot (tree_simple_ws)
    L.tree_off = off; off = align_up(off + (size_t)kMaxCh * 3 * kSteps * L.tree_slot, 4096);
    L.treell_slot = align_up(env_size("POLAR_TREELL_SLOT", 64 << 10), 512);
    L.treell_off = off; off = align_up(off + (size_t)kMaxCh * 3 * kSteps * L.treell_slot, 4096);
    L.os128_off = off; off = align_up(off + 2 * kMaxRanks * 2 * L.osll_chunk, 4096);
    L.ts128_off = off; off = align_up(off + 2 * (2 * kMaxRanks * 2 * L.tsll_chunk), 4096);
    L.ring128_slot = align_up(env_size("POLAR_RING128_SLOT", 128 << 10), 512);
    L.ring128_off = off; off = align_up(off + (size_t)kMaxCh * kSteps * L.ring128_slot, 4096);
    L.tree128_slot = align_up(env_size("POLAR_TREE128_SLOT", 64 << 10), 512);
    L.tree128_off = off; off = align_up(off + (size_t)kMaxCh * 3 * kSteps * L.tree128_slot, 4096);
    // two halves of 32 MiB: a 128 MiB message pipelines as 4 chunks
    L.bounce_bytes = with_bounce ? align_up(env_size("POLAR_BOUNCE", 64 << 20), 8192) : 0;
    L.bounce_off = off; off = align_up(off + L.bounce_bytes, 4096);
    L.probe_off = off; off = align_up(off + probe_ll128_region_bytes(kProbePairs), 4096);
    L.total = off;
    // NVLS: the region bound to the multicast object (real comms; every rank the same)
    L.nvls_bytes = with_bounce ? align_up(env_size("POLAR_NVLS_BYTES", 256 << 20), 2 << 20) : 0;
    {
        const char* e = std::getenv("POLAR_NVLS");
        if (e && e[0] == '0') L.nvls_bytes = 0;
    }
    return L;
}

}  // namespace polar

using namespace polar;

struct Registration {
    char* base;            // local device pointer
    size_t bytes;
    char* peer[kMaxRanks]; // rank p's registered base as mapped here
    char* peer_base[kMaxRanks];   // the IPC mapping (peer allocation start) behind peer[p]
    bool owned;            // allocated by polar_mem_alloc
    uint32_t id;           // registration sequence number (identical on every rank: collective)
    unsigned long long buffer_id;  // CU_POINTER_ATTRIBUTE_BUFFER_ID of the allocation at registration
};

struct polar_comm_s {
    int nranks = 0, rank0 = 0, nlocal = 0, device = 0;
    bool is_virtual = false;
    Layout L{};
    char* scratch_own[kMaxRanks] = {};   // allocations owned by this process
    char* scratch[kMaxRanks] = {};       // rank p's scratch as addressable here
    std::vector<Registration> regs;
    uint32_t reg_seq = 0;                // registrations made (collective, so equal on every rank)
    uint64_t stale_regs = 0;             // user registrations dropped because their allocation was freed
    std::vector<char*> ipc_mapped;       // to close at destroy
    // IPC handles already opened (one open per allocation).  peer_bid: the
    // peer's CU_POINTER_ATTRIBUTE_BUFFER_ID of that allocation when known (the
    // auto-registration exchange sends it; 0 from polar_register); last_use: the
    // auto-registration call that last used the mapping (0: never)
    struct Opened { int peer; cudaIpcMemHandle_t h; char* base; unsigned long long peer_bid; uint64_t last_use; };
    std::vector<Opened> opened;
    std::vector<char*> virt_allocs;      // polar_mem_alloc on virtual comms
    int* err_host = nullptr;
    int* err_dev = nullptr;
    polar_decision last{};
    uint32_t last_nch = 0;
    int last_transport = POLAR_TRANSPORT_PEER;
    uint64_t launches = 0;
    uint64_t calls = 0;                  // collective launches on this comm (identical on every rank)
    uint64_t prev_tag = 0;               // decision tag of the previous launch
    polar_status latched = POLAR_OK;
    polar_allgather_fn ag = nullptr;
    void* user = nullptr;
    uint64_t init_value = 0;
    int max_coop_blocks = 0;             // virtual: co-residency bound
    int share_cap = 0;                   // real comm with ranks sharing a GPU: channel cap (0: none)
    unsigned long long* trace = nullptr; // diagnostic per-CTA timestamps
    bool coop = true;                    // virtual: cooperative launch (co-residency guaranteed)
    bool pdl = true;                     // programmatic dependent launch (POLAR_PDL=0 disables)
    unsigned jitter_ns = 0;              // fault injection (POLAR_JITTER_NS)
    // profiler -> tuner closed loop (f3)
    Adaptive ad;
    TelEntry* tel_host = nullptr;        // host-mapped telemetry ring
    TelEntry* tel_dev = nullptr;
    unsigned long long tel_seq = 0;      // last launch sequence number handed out
    unsigned long long tel_consumed = 0; // samples consumed up to (and including) this seq
    int tma_mode = 2;                    // two-shot Simple via TMA smem staging: 0 never, 1 always, 2 auto
    int ring_tma = 0;                    // ring Simple via TMA-staged FIFOs (POLAR_RING_TMA=1 enables)
    size_t ring_tma_min = 0;             // ... from this many bytes per channel on (POLAR_RING_TMA_MIN)
    int ring_flags = 1;                  // ring_simple_tma: bit 0 L2 hints, bit 1 discard (POLAR_RING_TMA_FLAGS)
    unsigned long long timeout_ns = 0;
    // polar_allreduce_host chunk pipeline (created on first use)
    cudaStream_t hs_in = nullptr, hs_out = nullptr;
    // unregistered two-shot: copy-in / kernel / copy-out pipeline over the two
    // halves of the bounce region (created on first use)
    cudaStream_t bs_in = nullptr, bs_out = nullptr;
    bool bounce_full = false;            // POLAR_BOUNCE_FULL=1: bounce the own shard too (A/B)
    cudaEvent_t be_start = nullptr, be_in[2] = {}, be_k[2] = {}, be_out[2] = {};
    cudaEvent_t he_start = nullptr, he_in = nullptr, he_red = nullptr, he_out = nullptr;
    unsigned long long probe_epoch = 0;  // p2p probe calls (same count on every rank)
    NvlsState nvls;                      // switch reduction (f1): multicast object, if the node has one
    // LL128 rests on a warp's 128-B line store landing as one unit; a real comm
    // accepts LL128 only once polar_comm_probe_ll128 found no torn line over its
    // own transport (or POLAR_LL128_REAL=1 says so); virtual comms: one GPU,
    // probed by polar_probe_ll128 (profiles/r01_probe_ll128.jsonl)
    bool ll128_ok = true;
    // virtual comms: ring / tree Simple as thread-block clusters (cluster.cuh;
    // POLAR_CLUSTER=0 keeps the FIFO kernels); channel bound = clusters of n CTAs
    // that fit on the GPU at once (cudaOccupancyMaxActiveClusters)
    bool cluster = false;
    int cl_max_ch[5] = {};               // per algorithm id
    size_t cl_tree_max = ~(size_t)0;     // cluster tree up to this many bytes per rank (POLAR_CLUSTER_TREE_MAX)
    // auto-registration (polar_comm_autoreg): unregistered two-shot calls of at
    // least autoreg_min bytes exchange their buffers' IPC handles (one host
    // all-gather per call) and run zero-copy; the handles this rank exported,
    // by allocation (CU_POINTER_ATTRIBUTE_BUFFER_ID)
    size_t autoreg_min = ~(size_t)0;     // off
    struct Exported { unsigned long long bid; char* base; cudaIpcMemHandle_t h; };
    std::vector<Exported> exported;
    polar_autoreg_stats ar{};
    std::mutex mu;
};

namespace {

inline polar_status cuerr(cudaError_t e) { return e == cudaSuccess ? POLAR_OK : POLAR_ECUDA; }

// Make `dev` current for the scope and restore the caller's device on exit:
// no C-ABI entry point changes the calling thread's current device.
struct DeviceGuard {
    int prev = -1;
    bool ok = false;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        ok = (prev == dev) || cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

#define CU_TRY(x)                                   \
    do {                                            \
        cudaError_t _e = (x);                       \
        if (_e != cudaSuccess) return POLAR_ECUDA;  \
    } while (0)

int esize_of(int dtype) {
    switch (dtype) {
        case POLAR_INT32: case POLAR_FLOAT32: return 4;
        case POLAR_INT64: return 8;
        case POLAR_BFLOAT16: return 2;
    }
    return 0;
}

bool op_ok(int op) { return op == POLAR_SUM || op == POLAR_MAX || op == POLAR_MIN; }

void fill_params(const polar_comm_s* c, dev::Params& P) {
    std::memset(&P, 0, sizeof(P));
    for (int p = 0; p < c->nranks; ++p) P.scratch[p] = c->scratch[p];
    P.nranks = c->nranks;
    P.rank0 = c->rank0;
    P.err = c->err_dev;
    P.timeout_ns = c->timeout_ns;
    const Layout& L = c->L;
    P.flags_off = L.flags_off; P.state_off = L.state_off; P.tags_off = L.tags_off;
    P.os_off = L.os_off; P.os_chunk = L.os_chunk;
    P.osll_off = L.osll_off; P.osll_chunk = L.osll_chunk;
    P.tsll_off = L.tsll_off; P.tsll_chunk = L.tsll_chunk;
    P.ring_off = L.ring_off; P.ring_slot = L.ring_slot;
    P.ringll_off = L.ringll_off; P.ringll_slot = L.ringll_slot;
    P.tree_off = L.tree_off; P.tree_slot = L.tree_slot;
    P.treell_off = L.treell_off; P.treell_slot = L.treell_slot;
    P.os128_off = L.os128_off; P.ts128_off = L.ts128_off;
    P.ring128_off = L.ring128_off; P.ring128_slot = L.ring128_slot;
    P.tree128_off = L.tree128_off; P.tree128_slot = L.tree128_slot;
    P.trace = c->trace;
    P.sys = c->is_virtual ? 0 : 1;
    P.jitter_ns = c->jitter_ns;
}

polar_status check_latched(polar_comm_s* c) {
    if (c->latched != POLAR_OK) return c->latched;
    int e = *(volatile int*)c->err_host;
    if (e != 0) c->latched = (polar_status)e;
    return c->latched;
}

// Decision tag of one launch (SURVEY.md §8(b) "cross-rank consistency"): every
// field that must agree across ranks for the exchange to be correct.
// `path` identifies how the buffers are addressed (zero-copy registration id
// and offset, bounce, staged), so that ranks which took different paths for one
// call disagree in the tag.
constexpr uint64_t kPathBounce = 0xB0B0ull;   // two-shot through the scratch bounce region
constexpr uint64_t kPathNvls = 0x4E564Cull;    // NVLS through the multicast-bound region

uint64_t decision_tag(int kind, int algo, int proto, int nch, int dtype, int op, uint64_t count, int root,
                      uint64_t path = 0) {
    uint64_t h = ((uint64_t)kind) | ((uint64_t)algo << 4) | ((uint64_t)proto << 8) | ((uint64_t)nch << 12) |
                 ((uint64_t)dtype << 20) | ((uint64_t)op << 26) | ((uint64_t)(root & 0xff) << 30);
    h ^= count * 0x9E3779B97F4A7C15ull;
    h ^= (path + 0x632BE59BD9B4E019ull) * 0xD6E8FEB86659FD93ull;
    h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 29;
    return h | 1;   // never 0
}

polar_status launch_kernel(polar_comm_s* c, const void* fn, dev::Params& P, int grid, cudaStream_t stream,
                          size_t smem = 0) {
    // real comms: the kernel publishes P.dtag for launch P.call and checks the
    // peers' tags of the previous launch against P.prev_tag (kernels.cuh tag_begin/end)
    P.call = c->calls;
    P.prev_tag = c->prev_tag;
    void* args[] = {&P};
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(dev::kBlock);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attrs[2];
    unsigned n = 0;
    if (c->is_virtual && c->coop) {
        attrs[n].id = cudaLaunchAttributeCooperative;
        attrs[n].val.cooperative = 1;
        ++n;
    }
    if (c->pdl) {
        attrs[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attrs[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    cfg.attrs = attrs;
    cfg.numAttrs = n;
    cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
    if (e != cudaSuccess && c->pdl) {
        // PDL not accepted together with the other attributes here: disable it for this comm
        (void)cudaGetLastError();
        c->pdl = false;
        cfg.numAttrs = n - 1;
        e = cudaLaunchKernelExC(&cfg, fn, args);
    }
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        return POLAR_ECUDA;
    }
    c->launches++;
    c->calls++;
    c->prev_tag = P.dtag;
    return POLAR_OK;
}

// Cluster-transport kernels (virtual comms): grid = nch clusters of n CTAs,
// cluster rank = rank (cluster.cuh).  No cooperative attribute: a cluster's CTAs
// are co-scheduled by the hardware and channels never wait on each other.
polar_status launch_cluster(polar_comm_s* c, const void* fn, dev::Params& P, int algo, cudaStream_t stream) {
    P.call = c->calls;
    P.prev_tag = c->prev_tag;
    void* args[] = {&P};
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(P.nch * c->nranks));
    cfg.blockDim = dim3((unsigned)cluster_threads(algo));
    cfg.dynamicSmemBytes = cluster_smem_bytes(algo);
    cfg.stream = stream;
    cudaLaunchAttribute attrs[2];
    unsigned n = 0;
    attrs[n].id = cudaLaunchAttributeClusterDimension;
    attrs[n].val.clusterDim.x = (unsigned)c->nranks;
    attrs[n].val.clusterDim.y = 1;
    attrs[n].val.clusterDim.z = 1;
    ++n;
    if (c->pdl) {
        attrs[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attrs[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    cfg.attrs = attrs;
    cfg.numAttrs = n;
    cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
    if (e != cudaSuccess && c->pdl) {
        (void)cudaGetLastError();
        cfg.numAttrs = 1;
        e = cudaLaunchKernelExC(&cfg, fn, args);
    }
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        return POLAR_ECUDA;
    }
    c->launches++;
    c->calls++;
    c->prev_tag = P.dtag;
    return POLAR_OK;
}

// How many clusters of n CTAs of the algorithm's cluster kernel fit at once
// (0: the cluster path is unavailable for it).
int cluster_max_active(int algo, int nranks) {
    const void* fn = cluster_kernel_for(POLAR_FLOAT32, POLAR_SUM, algo);
    if (!fn) return 0;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(nranks * POLAR_MAXCH));
    cfg.blockDim = dim3((unsigned)cluster_threads(algo));
    cfg.dynamicSmemBytes = cluster_smem_bytes(algo);
    cudaLaunchAttribute a{};
    a.id = cudaLaunchAttributeClusterDimension;
    a.val.clusterDim.x = (unsigned)nranks;
    a.val.clusterDim.y = 1;
    a.val.clusterDim.z = 1;
    cfg.attrs = &a;
    cfg.numAttrs = 1;
    int num = 0;
    if (cudaOccupancyMaxActiveClusters(&num, fn, &cfg) != cudaSuccess) {
        (void)cudaGetLastError();
        return 0;
    }
    return num;
}

polar_status init_barrier(polar_comm_s* c) {
    dev::Params P;
    fill_params(c, P);
    P.nch = 1;
    c->init_value++;
    void* args[] = {&P, &c->init_value};
    cudaError_t e;
    if (c->is_virtual)
        e = cudaLaunchCooperativeKernel(init_barrier_kernel_ptr(), dim3(c->nlocal), dim3(dev::kBlock), args, 0, 0);
    else
        e = cudaLaunchKernel(init_barrier_kernel_ptr(), dim3(1), dim3(dev::kBlock), args, 0, 0);
    if (e != cudaSuccess) return POLAR_ECUDA;
    if (cudaDeviceSynchronize() != cudaSuccess) return POLAR_ECUDA;
    return check_latched(c);
}

polar_status alloc_common(polar_comm_s* c) {
    {
        const char* ev = std::getenv("POLAR_PDL");
        c->pdl = !(ev && ev[0] == '0');
        // TMA-staged two-shot: POLAR_TWOSHOT_TMA=1 always, =0 never, unset = auto:
        // virtual comms with n <= 4 and >= 64 MiB (measured, bf16 busBW at 1 GiB:
        // n=2 1103 vs 680, n=4 1247 vs 1170 GB/s; equal at n=8; LDG ahead below
        // 64 MiB, where the bulk pipeline fill costs ~8 us).  Real comms stay on LDG by default
        // until bulk copies over peer-mapped NVLink memory are validated on a
        // multi-GPU box (they are tested over same-GPU CUDA-IPC mappings).
        c->jitter_ns = (unsigned)env_size("POLAR_JITTER_NS", 0);
        const char* et = std::getenv("POLAR_TWOSHOT_TMA");
        c->tma_mode = et ? (et[0] == '1' ? 1 : 0) : 2;
        // TMA-staged ring Simple: opt-in (POLAR_RING_TMA=1).  On one GPU it is not
        // faster than the warp-specialised LDG ring (both sit at the memory-op
        // throughput of one HBM, DESIGN.md §8 "Ring on virtual ranks"), and bulk
        // copies over peer-mapped NVLink memory are not validated on this pool.
        const char* er = std::getenv("POLAR_RING_TMA");
        c->ring_tma = er && er[0] == '1';
        c->ring_tma_min = env_size("POLAR_RING_TMA_MIN", 0);
        {
            const char* eb = std::getenv("POLAR_BOUNCE_FULL");
            c->bounce_full = eb && eb[0] == '1';
        }
        {
            const char* ef = std::getenv("POLAR_RING_TMA_FLAGS");
            if (ef && *ef) c->ring_flags = (int)std::strtol(ef, nullptr, 0);
        }
    }
    // the two-shot Simple kernels may use up to tma_smem_bytes(8) of dynamic shared memory
    const int dts[] = {POLAR_INT32, POLAR_INT64, POLAR_FLOAT32, POLAR_BFLOAT16};
    const int ops[] = {POLAR_SUM, POLAR_MAX, POLAR_MIN};
    for (int dt : dts)
        for (int op : ops) {
            CU_TRY(cudaFuncSetAttribute(kernel_for(dt, op, POLAR_ALGO_TWOSHOT, POLAR_PROTO_SIMPLE),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)dev::tma_smem_bytes(kMaxRanks)));
            CU_TRY(cudaFuncSetAttribute(kernel_for(dt, op, POLAR_ALGO_RING, POLAR_PROTO_SIMPLE),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)dev::ring_tma_smem_bytes()));
            for (int algo : {POLAR_ALGO_RING, POLAR_ALGO_TREE})
                if (const void* fn = cluster_kernel_for(dt, op, algo))
                    CU_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)cluster_smem_bytes(algo)));
        }
    c->timeout_ns = (unsigned long long)env_size("POLAR_TIMEOUT_MS", 20000) * 1000000ull;
    CU_TRY(cudaHostAlloc(reinterpret_cast<void**>(&c->err_host), sizeof(int), cudaHostAllocMapped));
    *c->err_host = 0;
    CU_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->err_dev), c->err_host, 0));
    CU_TRY(cudaHostAlloc(reinterpret_cast<void**>(&c->tel_host), sizeof(TelEntry) * kTelRing, cudaHostAllocMapped));
    std::memset(c->tel_host, 0, sizeof(TelEntry) * kTelRing);
    CU_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->tel_dev), c->tel_host, 0));
    {
        polar_adaptive_params p{};
        p.enabled = 0;
        p.period = 1000;
        p.c_min = 2;
        p.contention_factor = 4.0;
        p.latency_scale = 1.0;
        adaptive_reset(c->ad, p);
    }
    return POLAR_OK;
}

// Driver entry points through the runtime (no -lcuda link).
template <class F> F driver_fn(const char* name) {
    cudaDriverEntryPointQueryResult q;
    void* fp = nullptr;
    if (cudaGetDriverEntryPoint(name, &fp, cudaEnableDefault, &q) != cudaSuccess || !fp) return nullptr;
    return reinterpret_cast<F>(fp);
}

// Drop registration i: close every peer IPC mapping no other registration uses
// (a peer allocation may back several registrations: caching allocators).
void release_registration(polar_comm_s* c, size_t i) {
    const Registration r = c->regs[i];
    c->regs.erase(c->regs.begin() + (long)i);
    for (int p = 0; p < c->nranks; ++p) {
        char* b = r.peer_base[p];
        if (p == c->rank0 || !b) continue;
        bool used = false;
        for (const auto& o : c->regs) used = used || o.peer_base[p] == b;
        if (used) continue;
        for (size_t k = 0; k < c->opened.size(); ++k)
            if (c->opened[k].peer == p && c->opened[k].base == b) {
                cudaIpcCloseMemHandle(b);
                c->opened.erase(c->opened.begin() + (long)k);
                break;
            }
        for (size_t m = 0; m < c->ipc_mapped.size(); ++m)
            if (c->ipc_mapped[m] == b) {
                c->ipc_mapped.erase(c->ipc_mapped.begin() + (long)m);
                break;
            }
    }
}

// Unique id of the allocation containing p (never reused within a process:
// CU_POINTER_ATTRIBUTE_BUFFER_ID), 0 if unknown.
unsigned long long buffer_id_of(const void* p) {
    using Fn = CUresult (*)(void*, CUpointer_attribute, CUdeviceptr);
    static Fn get = driver_fn<Fn>("cuPointerGetAttribute");
    unsigned long long id = 0;
    if (!get || get(&id, CU_POINTER_ATTRIBUTE_BUFFER_ID, (CUdeviceptr)p) != CUDA_SUCCESS) return 0;
    return id;
}

// find a registration containing [p, p+bytes).  A user registration whose
// allocation was freed since (a caching allocator may hand the same addresses
// to a new allocation, which peers' IPC mappings do not show) is stale: it is
// dropped here, and the call takes the path of an unregistered buffer.  The
// decision tag carries the path and the registration id, so ranks that disagree
// are caught by the entry handshake before any data moves.
const Registration* find_reg(polar_comm_s* c, const char* p, size_t bytes) {
    for (size_t i = 0; i < c->regs.size(); ++i) {
        const Registration& r = c->regs[i];
        if (!(p >= r.base && p + bytes <= r.base + r.bytes)) continue;
        if (!r.owned && r.buffer_id && buffer_id_of(p) != r.buffer_id) {
            release_registration(c, i);   // local: closes this rank's mappings of the peers' buffers
            c->stale_regs++;
            return nullptr;
        }
        return &c->regs[i];
    }
    return nullptr;
}

// Host barrier over the bootstrap all-gather (real comms): every rank's device
// work has completed before anyone unmaps or frees memory a peer may still be
// touching (a final credit or exit flag posted into my scratch after my kernel
// returned, for example).
polar_status host_barrier(polar_comm_s* c) {
    if (c->is_virtual || c->nranks == 1 || !c->ag) return POLAR_OK;
    uint64_t mine = 0x62617272ull, all[kMaxRanks];
    return c->ag(&mine, all, sizeof(uint64_t), c->user) == 0 ? POLAR_OK : POLAR_ESTATE;
}

void destroy_comm(polar_comm_s* c, bool collective) {
    if (!c) return;
    DeviceGuard dg(c->device);
    cudaDeviceSynchronize();
    if (collective) (void)host_barrier(c);
    nvls_teardown(c->nvls, c->device);
    for (char* m : c->ipc_mapped) cudaIpcCloseMemHandle(m);
    for (auto& r : c->regs)
        if (r.owned) cudaFree(r.base);
    for (char* v : c->virt_allocs) cudaFree(v);
    for (int p = 0; p < kMaxRanks; ++p)
        if (c->scratch_own[p]) cudaFree(c->scratch_own[p]);
    if (c->err_host) cudaFreeHost(c->err_host);
    if (c->tel_host) cudaFreeHost(c->tel_host);
    if (c->hs_in) cudaStreamDestroy(c->hs_in);
    if (c->hs_out) cudaStreamDestroy(c->hs_out);
    if (c->bs_in) cudaStreamDestroy(c->bs_in);
    if (c->bs_out) cudaStreamDestroy(c->bs_out);
    for (cudaEvent_t e : {c->be_start, c->be_in[0], c->be_in[1], c->be_k[0], c->be_k[1], c->be_out[0], c->be_out[1]})
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : {c->he_start, c->he_in, c->he_red, c->he_out})
        if (e) cudaEventDestroy(e);
    delete c;
}

// The allocation containing p: cuMemGetAddressRange through the runtime's
// driver entry point (no -lcuda link).  false if unknown.
bool alloc_range(const void* p, char** base, size_t* bytes) {
    static CUresult (*getrange)(CUdeviceptr*, size_t*, CUdeviceptr) = nullptr;
    if (!getrange) {
        cudaDriverEntryPointQueryResult q;
        void* fp = nullptr;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fp, cudaEnableDefault, &q) != cudaSuccess || !fp)
            return false;
        getrange = reinterpret_cast<CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr)>(fp);
    }
    CUdeviceptr b = 0;
    size_t sz = 0;
    if (getrange(&b, &sz, (CUdeviceptr)p) != CUDA_SUCCESS) return false;
    *base = reinterpret_cast<char*>(b);
    *bytes = sz;
    return true;
}

// Exchange IPC handles of `base` (allocation start) + offset; fill peer[] pointers.
polar_status exchange_and_map(polar_comm_s* c, char* ptr, char* peer[kMaxRanks], char* peer_base[kMaxRanks] = nullptr) {
    struct Msg { cudaIpcMemHandle_t h; unsigned long long off; int pid_ok; };
    char* base = nullptr;
    size_t sz = 0;
    if (!alloc_range(ptr, &base, &sz)) return POLAR_EINVAL;
    Msg mine{};
    CU_TRY(cudaIpcGetMemHandle(&mine.h, reinterpret_cast<void*>(base)));
    mine.off = (unsigned long long)(ptr - base);
    mine.pid_ok = 1;
    std::vector<Msg> all(c->nranks);
    if (c->ag(&mine, all.data(), sizeof(Msg), c->user) != 0) return POLAR_ESTATE;
    for (int p = 0; p < c->nranks; ++p) {
        if (peer_base) peer_base[p] = nullptr;
        if (p == c->rank0) { peer[p] = ptr; continue; }
        // a peer allocation may back several registrations (caching allocators):
        // open each IPC handle once and reuse the mapping
        char* base_p = nullptr;
        for (const auto& o : c->opened)
            if (o.peer == p && std::memcmp(&o.h, &all[p].h, sizeof(cudaIpcMemHandle_t)) == 0) base_p = o.base;
        if (!base_p) {
            void* m = nullptr;
            cudaError_t e = cudaIpcOpenMemHandle(&m, all[p].h, cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) { (void)cudaGetLastError(); return POLAR_ECUDA; }
            base_p = reinterpret_cast<char*>(m);
            c->ipc_mapped.push_back(base_p);
            c->opened.push_back({p, all[p].h, base_p, 0ull, 0});
        }
        peer[p] = base_p + all[p].off;
        if (peer_base) peer_base[p] = base_p;
    }
    return POLAR_OK;
}

// ------------------------------------------------------- auto-registration
// polar_comm_autoreg (DESIGN.md §8 "Unregistered buffers: auto-registration").
// An unregistered two-shot call of at least autoreg_min bytes: every rank sends
// {IPC handle of the allocation holding its buffer, that allocation's buffer
// id, the buffer's offset in it, the call's bytes, ok}; every rank maps the
// peers' allocations (cached per (peer, handle, buffer id): the first call on
// an allocation opens it, later calls only exchange) and addresses peer p's
// buffer as its mapping + offset_p, so offsets may differ between ranks.  Zero
// copy or bounce is decided from the gathered records alone, hence the same on
// every rank; a rank whose buffer is not IPC-exportable (cuMem / VMM memory)
// sends ok = 0 and every rank bounces.  The path hash (buffer ids and offsets
// of all ranks) goes into the decision tag.
constexpr size_t kAutoExported = 64;   // exported handles remembered (per comm)
constexpr size_t kAutoMapped = 32;     // auto-opened peer mappings kept per peer
constexpr uint64_t kPathAuto = 0xA0705E6ull;

struct AutoMsg {
    cudaIpcMemHandle_t h;
    unsigned long long bid, off, bytes, dtag;
    uint32_t ok, pad;
};

// close mapping k of c->opened (no registration uses it); the device is
// synchronised first: a kernel of mine still in flight may address it
void close_opened(polar_comm_s* c, size_t k) {
    cudaDeviceSynchronize();
    char* b = c->opened[k].base;
    cudaIpcCloseMemHandle(b);
    c->opened.erase(c->opened.begin() + (long)k);
    for (size_t m = 0; m < c->ipc_mapped.size(); ++m)
        if (c->ipc_mapped[m] == b) {
            c->ipc_mapped.erase(c->ipc_mapped.begin() + (long)m);
            break;
        }
    c->ar.evictions++;
}

bool used_by_registration(const polar_comm_s* c, int p, const char* b) {
    for (const auto& r : c->regs)
        if (r.peer_base[p] == b) return true;
    return false;
}

// The exchange runs for every call of >= autoreg_min bytes on a real comm,
// whatever this rank's decision or registrations: the call sequence (and so the
// exchange count) is the same on every rank even when the ranks' policies or
// registrations disagree, and the record carries the decision tag, so such a
// disagreement is caught here, synchronously, on every rank (ESTATE latched,
// nothing launched) instead of leaving one rank blocked in the all-gather.
// map = the decision is two-shot Simple: *zc = true: ptrs[] hold every rank's
// buffer as addressable here, *path the tag component; *zc = false: bounce
// (every rank agrees).  ECUDA if a peer's handle cannot be opened.
polar_status autoreg_map(polar_comm_s* c, char* mine, size_t bytes, uint64_t dtag, bool map, cudaStream_t stream,
                         char* ptrs[kMaxRanks], uint64_t* path, bool* zc) {
    *zc = false;
    AutoMsg m{};
    m.bytes = bytes;
    m.dtag = dtag;
    char* base = nullptr;
    size_t sz = 0;
    const unsigned long long bid = buffer_id_of(mine);
    if (bid && alloc_range(mine, &base, &sz) && mine + bytes <= base + sz) {
        int e = -1;
        for (size_t i = 0; i < c->exported.size(); ++i)
            if (c->exported[i].bid == bid && c->exported[i].base == base) e = (int)i;
        if (e < 0) {
            polar_comm_s::Exported x{bid, base, {}};
            if (cudaIpcGetMemHandle(&x.h, base) == cudaSuccess) {
                if (c->exported.size() >= kAutoExported) c->exported.erase(c->exported.begin());
                c->exported.push_back(x);
                e = (int)c->exported.size() - 1;
            } else {
                (void)cudaGetLastError();
            }
        }
        if (e >= 0) {
            m.h = c->exported[(size_t)e].h;
            m.bid = bid;
            m.off = (unsigned long long)(mine - base);
            m.ok = 1;
        }
    }
    std::vector<AutoMsg> all(c->nranks);
    c->ar.exchanges++;
    if (c->ag(&m, all.data(), sizeof(AutoMsg), c->user) != 0) return POLAR_ESTATE;
    bool ok = true;
    uint64_t h = 0xcbf29ce484222325ull;
    for (int p = 0; p < c->nranks; ++p) {
        if (all[p].dtag != dtag || all[p].bytes != bytes) {
            c->latched = POLAR_ESTATE;   // the ranks decided this call differently
            c->ar.mismatches++;
            return POLAR_ESTATE;
        }
        ok = ok && all[p].ok;
        h = (h ^ all[p].bid) * 0x100000001B3ull;
        h = (h ^ all[p].off) * 0x100000001B3ull;
    }
    if (!map) return POLAR_OK;
    if (!ok) {
        c->ar.bounced++;
        return POLAR_OK;
    }
    // no device synchronise (eviction) while the caller's stream is being captured
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    const bool capturing = cudaStreamIsCapturing(stream, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone;
    const uint64_t use = c->ar.exchanges;
    for (int p = 0; p < c->nranks; ++p) {
        if (p == c->rank0) {
            ptrs[p] = mine;
            continue;
        }
        long k = -1;
        for (size_t i = 0; i < c->opened.size(); ++i)
            if (c->opened[i].peer == p && std::memcmp(&c->opened[i].h, &all[p].h, sizeof(cudaIpcMemHandle_t)) == 0) {
                k = (long)i;
                break;
            }
        if (k >= 0 && c->opened[(size_t)k].peer_bid && c->opened[(size_t)k].peer_bid != all[p].bid) {
            // the same handle for another allocation of the peer (freed and
            // re-allocated): the mapping is stale
            if (used_by_registration(c, p, c->opened[(size_t)k].base) || capturing) return POLAR_ESTATE;
            close_opened(c, (size_t)k);
            k = -1;
        }
        if (k < 0) {
            // bound the auto-opened mappings of this peer: drop the least recently used
            size_t nmap = 0, lru = 0;
            uint64_t oldest = ~0ull;
            for (size_t i = 0; i < c->opened.size(); ++i) {
                const auto& o = c->opened[i];
                if (o.peer != p || o.last_use == 0 || used_by_registration(c, p, o.base)) continue;
                ++nmap;
                if (o.last_use < oldest && o.last_use != use) { oldest = o.last_use; lru = i; }
            }
            if (nmap >= kAutoMapped && oldest != ~0ull && !capturing) close_opened(c, lru);
            void* mp = nullptr;
            if (cudaIpcOpenMemHandle(&mp, all[p].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                (void)cudaGetLastError();
                return POLAR_ECUDA;
            }
            c->ipc_mapped.push_back(reinterpret_cast<char*>(mp));
            c->opened.push_back({p, all[p].h, reinterpret_cast<char*>(mp), all[p].bid, use});
            c->ar.opens++;
            k = (long)c->opened.size() - 1;
        }
        auto& o = c->opened[(size_t)k];
        o.peer_bid = all[p].bid;
        o.last_use = use;
        ptrs[p] = o.base + all[p].off;
    }
    *path = h;
    *zc = true;
    c->ar.zero_copy++;
    return POLAR_OK;
}

// Co-residency bound of a launch on one device: SMs x the fewest CTAs per SM
// of any AllReduce kernel we may launch (virtual comms clamp their grids to it;
// real comms whose ranks share a GPU divide it among those ranks).
polar_status coresident_blocks(int cuda_device, int* blocks) {
    int sms = 0, per_sm = 0, minper = 1 << 30;
    polar_status st = cuerr(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cuda_device));
    const int dts[] = {POLAR_INT32, POLAR_INT64, POLAR_FLOAT32, POLAR_BFLOAT16};
    const int ops[] = {POLAR_SUM, POLAR_MAX, POLAR_MIN};
    const int algos[] = {POLAR_ALGO_TREE, POLAR_ALGO_RING, POLAR_ALGO_ONESHOT, POLAR_ALGO_TWOSHOT};
    const int protos[] = {POLAR_PROTO_LL, POLAR_PROTO_LL128, POLAR_PROTO_SIMPLE};
    for (int dt : dts) for (int op : ops) for (int a : algos) for (int pr : protos) {
        if (st != POLAR_OK) break;
        const void* fn = kernel_for(dt, op, a, pr);
        st = cuerr(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, dev::kBlock, 0));
        minper = std::min(minper, per_sm);
    }
    *blocks = sms * minper;
    return st;
}

struct BootRec {
    uint64_t magic;
    uint32_t nranks, rank;
    uint64_t layout_hash;
    uint64_t pad;
    unsigned char uuid[16];   // the rank's GPU (zeros from polar_bootstrap_check)
};
static_assert(sizeof(BootRec) == 48, "bootstrap record is 48 B");
constexpr uint64_t kBootMagic = 0x706f6c6172763031ull;   // "polarv01"

uint64_t layout_hash(const Layout& L) {
    // FNV-1a over the layout (every offset/size must match across ranks)
    const unsigned char* p = reinterpret_cast<const unsigned char*>(&L);
    uint64_t h = 1469598103934665603ull;
    for (size_t i = 0; i < sizeof(Layout); ++i) { h ^= p[i]; h *= 1099511628211ull; }
    return h;
}

// uuid: this rank's GPU (may be null); *shared_gpu (may be null) is set when
// another rank reports the same GPU (several ranks on one device, e.g. MPS).
polar_status bootstrap_check(int nranks, int rank, const Layout& L, polar_allgather_fn ag, void* user,
                             const unsigned char* uuid = nullptr, bool* shared_gpu = nullptr,
                             int* max_per_gpu = nullptr) {
    BootRec mine{kBootMagic, (uint32_t)nranks, (uint32_t)rank, layout_hash(L), 0, {}};
    if (uuid) std::memcpy(mine.uuid, uuid, sizeof(mine.uuid));
    std::vector<BootRec> all(nranks);
    if (ag(&mine, all.data(), sizeof(BootRec), user) != 0) return POLAR_ESTATE;
    bool shared = false;
    for (int p = 0; p < nranks; ++p) {
        const BootRec& r = all[p];
        if (r.magic != kBootMagic || r.nranks != (uint32_t)nranks || r.rank != (uint32_t)p ||
            r.layout_hash != mine.layout_hash)
            return POLAR_ESTATE;
        if (p != rank && std::memcmp(r.uuid, mine.uuid, sizeof(mine.uuid)) == 0) shared = true;
    }
    if (shared_gpu) *shared_gpu = shared;
    if (max_per_gpu) {
        // the most ranks any one GPU hosts (the same on every rank: gathered data)
        int most = 1;
        for (int p = 0; p < nranks; ++p) {
            int k = 0;
            for (int q = 0; q < nranks; ++q) k += std::memcmp(all[p].uuid, all[q].uuid, sizeof(mine.uuid)) == 0;
            most = std::max(most, k);
        }
        *max_per_gpu = most;
    }
    return POLAR_OK;
}

// Profiler side: fold every completed telemetry sample since the last drain
// into the open window (latency_scale applied: contention injection).
void adaptive_drain(polar_comm_s* c) {
    while (c->tel_consumed < c->tel_seq) {
        const unsigned long long want = c->tel_consumed + 1;
        volatile TelEntry* e = c->tel_host + (want % kTelRing);
        const unsigned long long seq = e->seq;
        if (seq < want) break;                       // not completed yet (or never written)
        if (seq == want) {
            const double ns = (double)(e->t1 - e->t0) * c->ad.prm.latency_scale;
            c->ad.win_sum += ns;
            c->ad.win_cnt++;
            c->ad.samples++;
        }                                            // seq > want: overwritten by a later lap, lost
        c->tel_consumed = want;
    }
}

// Tuner side: at every `period`-th adaptive call (the same call index on every
// rank) close the window.  Real comms gather the window means of all ranks
// through the bootstrap all-gather and use their max, so every rank applies the
// same rule to the same number and launches the same channel count.
polar_status adaptive_tick(polar_comm_s* c, uint32_t cap) {
    Adaptive& a = c->ad;
    a.calls++;
    if (a.calls % a.prm.period != 0) return POLAR_OK;
    adaptive_drain(c);
    double m = a.win_cnt ? a.win_sum / (double)a.win_cnt : 0.0;
    if (!c->is_virtual && c->nranks > 1) {
        std::vector<double> all(c->nranks, 0.0);
        if (c->ag(&m, all.data(), sizeof(double), c->user) != 0) return POLAR_ESTATE;
        m = 0.0;
        for (double x : all) m = x > m ? x : m;
    }
    adaptive_close_window(a, m, cap);
    a.win_sum = 0.0;
    a.win_cnt = 0;
    return POLAR_OK;
}

polar_status do_allreduce(polar_comm_s* c, void* const* bufs, size_t count, int dtype, int op,
                          const polar_decision* forced, cudaStream_t stream) {
    const int es = esize_of(dtype);
    if (!es || !op_ok(op)) return POLAR_EINVAL;
    if (count > 0 && !bufs) return POLAR_EINVAL;
    for (int l = 0; l < c->nlocal && count > 0; ++l)
        if (!bufs[l] || (reinterpret_cast<uintptr_t>(bufs[l]) % es) != 0) return POLAR_EINVAL;
    polar_status st = check_latched(c);
    if (st != POLAR_OK) return st;
    // --- decide (the tuner hook)
    polar_decision d;
    polar_ctx ctx{POLAR_COLL_ALLREDUCE, (uint32_t)c->nranks, (uint64_t)count * (uint64_t)es};
    if (forced) {
        d = *forced;
        if (d.nchannels < 1) d.nchannels = 1;
        if (d.nchannels > POLAR_MAXCH) d.nchannels = POLAR_MAXCH;
        d.generation = polar_policy_generation();
    } else {
        st = polar_decide(&ctx, &d);
        if (st != POLAR_OK) return st;
    }
    const bool nvls = d.algo == POLAR_ALGO_NVLS;
    const void* fn = nvls ? (c->nvls.ok ? nvls_kernel_for(dtype, op) : nullptr)
                          : kernel_for(dtype, op, (int)d.algo, (int)d.proto);
    if (!fn) return POLAR_EUNSUPPORTED;
    if (d.proto == POLAR_PROTO_LL128 && !c->ll128_ok) return POLAR_EUNSUPPORTED;   // premise not probed here
    c->last = d;                      // the policy's decision (what the hook returned)
    const bool adaptive_row = (d.flags & POLAR_ROW_ADAPTIVE_NCH) && count > 0 && c->nranks > 1;
    if (c->ad.prm.enabled && count > 0 && c->nranks > 1) {
        // The window schedule counts every AllReduce of the comm while the loop is
        // enabled (polar_adaptive_config is collective), never the local policy:
        // a rank whose table differs cannot leave its peers blocked in the
        // window all-gather of a real comm.  The cap is the last adaptive row's.
        if (adaptive_row) c->ad.cap = d.nchannels;
        st = adaptive_tick(c, c->ad.cap);
        if (st != POLAR_OK) return st;
    }
    if (adaptive_row) {
        // closed loop: the row's nchannels is the cap, the controller picks c
        d.nchannels = c->ad.c < d.nchannels ? c->ad.c : d.nchannels;
    }
    // virtual comms: ring / tree Simple on whole 16-B packs of 16-B aligned
    // buffers run as clusters (cluster.cuh), bounded by the clusters that fit
    bool use_cluster = false;
    if (c->is_virtual && c->cluster && d.proto == POLAR_PROTO_SIMPLE &&
        (d.algo == POLAR_ALGO_RING || d.algo == POLAR_ALGO_TREE) &&
        c->cl_max_ch[d.algo] > 0 && (count * (size_t)es) % 16 == 0 &&
        (d.algo == POLAR_ALGO_RING || count * (size_t)es <= c->cl_tree_max)) {
        use_cluster = true;
        for (int p = 0; p < c->nranks && count > 0; ++p)
            use_cluster = use_cluster && (reinterpret_cast<uintptr_t>(bufs[p]) % 16 == 0);
        use_cluster = use_cluster && cluster_kernel_for(dtype, op, (int)d.algo) != nullptr;
    }
    if (use_cluster) {
        if ((int)d.nchannels > c->cl_max_ch[d.algo]) d.nchannels = (uint32_t)c->cl_max_ch[d.algo];
    } else if (c->is_virtual) {
        const int maxch = std::max(1, c->max_coop_blocks / c->nranks);
        if ((int)d.nchannels > maxch) d.nchannels = (uint32_t)maxch;   // co-residency bound
    } else if (c->share_cap > 0 && (int)d.nchannels > c->share_cap) {
        d.nchannels = (uint32_t)c->share_cap;                          // ranks sharing a GPU
    }
    c->last_nch = d.nchannels;        // what is launched
    c->last_transport = use_cluster ? POLAR_TRANSPORT_CLUSTER : POLAR_TRANSPORT_PEER;
    if (count == 0 || c->nranks == 1) return POLAR_OK;
    DeviceGuard dg(c->device);
    if (!dg.ok) return POLAR_ECUDA;

    dev::Params P;
    fill_params(c, P);
    P.nch = (int)d.nchannels;
    const int grid = c->nlocal * P.nch;
    // the bounce path launches per chunk: each launch's count is in its own tag
    P.dtag = decision_tag(0, (int)d.algo, (int)d.proto, P.nch, dtype, op, count, 0);
    if (c->ad.prm.enabled && adaptive_row) {
        // telemetry from adaptive-row launches only: a window's mean never mixes
        // in the latencies of other sizes or algorithms
        adaptive_drain(c);           // keep the ring from lapping between windows
        P.tel = c->tel_dev;
        P.seq = ++c->tel_seq;
    }
    const bool ts_simple = d.algo == POLAR_ALGO_TWOSHOT && d.proto == POLAR_PROTO_SIMPLE;
    const bool tma_auto = c->is_virtual && c->nranks <= 4 && count * (size_t)es >= (64u << 20);
    P.tma = (ts_simple && (c->tma_mode == 1 || (c->tma_mode == 2 && tma_auto))) ? 1 : 0;
    const bool ring_simple = d.algo == POLAR_ALGO_RING && d.proto == POLAR_PROTO_SIMPLE;
    P.ring_tma = (ring_simple && c->ring_tma && count * (size_t)es / d.nchannels >= c->ring_tma_min) ? 1 : 0;
    P.ring_flags = c->ring_flags;
    const size_t smem = P.tma ? dev::tma_smem_bytes(c->nranks) : (P.ring_tma ? dev::ring_tma_smem_bytes() : 0);
    const size_t bytes = count * (size_t)es;

    if (c->is_virtual) {
        bool vec = true;
        for (int p = 0; p < c->nranks; ++p) {
            P.bufs[p] = reinterpret_cast<char*>(bufs[p]);
            vec = vec && (reinterpret_cast<uintptr_t>(bufs[p]) % 16 == 0);
        }
        P.vec = vec;
        P.count = count;
        if (use_cluster) return launch_cluster(c, cluster_kernel_for(dtype, op, (int)d.algo), P, (int)d.algo, stream);
        return launch_kernel(c, fn, P, grid, stream, smem);
    }
    char* mine = reinterpret_cast<char*>(bufs[0]);
    // auto-registration: one exchange per call of >= autoreg_min bytes, before
    // any path choice (it is also the synchronous decision check)
    const bool ar_on = bytes >= c->autoreg_min && c->ag != nullptr;
    bool ar_zc = false;
    char* ar_ptrs[kMaxRanks] = {};
    uint64_t ar_path = 0;
    if (ar_on) {
        st = autoreg_map(c, mine, bytes, P.dtag, ts_simple, stream, ar_ptrs, &ar_path, &ar_zc);
        if (st != POLAR_OK) return st;
    }
    if (nvls) {
        // switch reduction over the bound region (nvls.cu): every rank copies its
        // input in, the kernel reduces through the multicast mapping, every rank
        // copies the result out; chunked by the region (minus one pad pack)
        const size_t chunk_elems = std::max<size_t>(16 / es, ((c->nvls.bytes - 16) / es) / (16 / es) * (16 / es));
        P.bufs[c->rank0] = c->nvls.uc;
        P.recv[0] = c->nvls.mc;
        P.vec = 1;
        for (size_t done = 0; done < count; done += chunk_elems) {
            const size_t n = std::min(chunk_elems, count - done);
            char* src = mine + done * es;
            CU_TRY(cudaMemcpyAsync(c->nvls.uc, src, n * es, cudaMemcpyDeviceToDevice, stream));
            P.count = n;
            P.dtag = decision_tag(0, (int)d.algo, (int)d.proto, P.nch, dtype, op, n, 0, kPathNvls);
            st = launch_kernel(c, fn, P, grid, stream, 0);
            if (st != POLAR_OK) return st;
            CU_TRY(cudaMemcpyAsync(src, c->nvls.uc, n * es, cudaMemcpyDeviceToDevice, stream));
        }
        return POLAR_OK;
    }
    if (d.algo != POLAR_ALGO_TWOSHOT || d.proto != POLAR_PROTO_SIMPLE) {
        // only the local buffer is touched directly; peers go through scratch
        P.bufs[c->rank0] = mine;
        P.vec = reinterpret_cast<uintptr_t>(mine) % 16 == 0;
        P.count = count;
        return launch_kernel(c, fn, P, grid, stream, smem);
    }
    // zero-copy two-shot needs every rank's buffer mapped
    if (ar_zc) {
        // auto-registered: every rank's buffer at its own offset
        bool vec = true;
        for (int p = 0; p < c->nranks; ++p) {
            P.bufs[p] = ar_ptrs[p];
            vec = vec && (reinterpret_cast<uintptr_t>(ar_ptrs[p]) % 16 == 0);
        }
        P.vec = vec;
        P.count = count;
        P.dtag = decision_tag(0, (int)d.algo, (int)d.proto, P.nch, dtype, op, count, 0, kPathAuto ^ ar_path);
        return launch_kernel(c, fn, P, grid, stream, smem);
    }
    // (with auto-registration on and some rank's buffer not exportable, every
    // rank bounces, registered or not: the gathered records decided it)
    const Registration* reg = ar_on ? nullptr : find_reg(c, mine, bytes);
    if (reg) {
        const size_t off = (size_t)(mine - reg->base);
        bool vec = true;
        for (int p = 0; p < c->nranks; ++p) {
            P.bufs[p] = reg->peer[p] + off;
            vec = vec && (reinterpret_cast<uintptr_t>(P.bufs[p]) % 16 == 0);
        }
        P.vec = vec;
        P.count = count;
        // zero-copy: every rank must address the same registration at the same offset
        P.dtag = decision_tag(0, (int)d.algo, (int)d.proto, P.nch, dtype, op, count, 0,
                              ((uint64_t)(reg->id + 1) << 40) ^ (uint64_t)off);
        return launch_kernel(c, fn, P, grid, stream, smem);
    }
    // Unregistered buffer: its peers cannot address it, so it travels through
    // the symmetric bounce region, split in two halves that alternate by chunk.
    // Copy-in of chunk k+1 (library stream bs_in), the two-shot kernel of chunk
    // k (the caller's stream) and copy-out of chunk k-1 (bs_out) overlap; over
    // NVLink the local copies hide behind the NVLink-bound kernel.  Half h is
    // refilled only after the copy-out of the chunk before (which followed its
    // kernel, whose exit barrier means no peer still reads it).  The caller's
    // stream waits for the last copy-out, so stream order is kept for the user.
    if (!c->bs_in) {
        CU_TRY(cudaStreamCreateWithFlags(&c->bs_in, cudaStreamNonBlocking));
        CU_TRY(cudaStreamCreateWithFlags(&c->bs_out, cudaStreamNonBlocking));
        CU_TRY(cudaEventCreateWithFlags(&c->be_start, cudaEventDisableTiming));
        for (int h = 0; h < 2; ++h) {
            CU_TRY(cudaEventCreateWithFlags(&c->be_in[h], cudaEventDisableTiming));
            CU_TRY(cudaEventCreateWithFlags(&c->be_k[h], cudaEventDisableTiming));
            CU_TRY(cudaEventCreateWithFlags(&c->be_out[h], cudaEventDisableTiming));
        }
    }
    const size_t half = (c->L.bounce_bytes / 2) & ~(size_t)15;
    const size_t chunk_elems = std::max<size_t>(16 / es, (half / es) / (16 / es) * (16 / es));
    P.vec = 1;   // the bounce halves are 16-B aligned on every rank
    // My own shard never needs the bounce: as its owner I read it from the user
    // buffer and store its result there (P.bufs[rank0] = the user buffer); only
    // the shards my peers own travel through my bounce half — copied in, reduced
    // by their owners in place, copied out.  That saves 2 · S/n of local copies
    // per call (half of them at n = 2).  Needs a 16-B aligned user buffer (the
    // kernel's fast path); otherwise the whole chunk bounces.
    const bool own_direct = (reinterpret_cast<uintptr_t>(mine) % 16 == 0) && !c->bounce_full;
    const size_t V = 16 / (size_t)es;
    CU_TRY(cudaEventRecord(c->be_start, stream));
    CU_TRY(cudaStreamWaitEvent(c->bs_in, c->be_start, 0));
    CU_TRY(cudaStreamWaitEvent(c->bs_out, c->be_start, 0));
    size_t k = 0;
    for (size_t done = 0; done < count; done += chunk_elems, ++k) {
        const int h = (int)(k & 1);
        const size_t n = std::min(chunk_elems, count - done);
        char* src = mine + done * es;
        for (int p = 0; p < c->nranks; ++p) P.bufs[p] = c->scratch[p] + c->L.bounce_off + (size_t)h * half;
        char* bnc = P.bufs[c->rank0];
        // my shard of this chunk, in elements: the kernel's split (kernels.cuh
        // twoshot_geo: split_range over 32-pack units)
        size_t e0 = 0, e1 = 0;
        if (own_direct) {
            const size_t np = (n + V - 1) / V, units = (np + 31) / 32;
            const size_t ua = units * (size_t)c->rank0 / (size_t)c->nranks;
            const size_t ub = units * (size_t)(c->rank0 + 1) / (size_t)c->nranks;
            e0 = std::min(n, ua * 32 * V);
            e1 = std::min(n, ub * 32 * V);
            P.bufs[c->rank0] = src;
        }
        auto copy_others = [&](char* dst, const char* from, cudaStream_t s) -> cudaError_t {
            // everything but [e0, e1) (own_direct), else the whole chunk
            cudaError_t e = cudaSuccess;
            if (e0 > 0) e = cudaMemcpyAsync(dst, from, e0 * es, cudaMemcpyDeviceToDevice, s);
            if (e == cudaSuccess && e1 < n)
                e = cudaMemcpyAsync(dst + e1 * es, from + e1 * es, (n - e1) * es, cudaMemcpyDeviceToDevice, s);
            return e;
        };
        if (!own_direct) e1 = 0;   // [e0, e1) empty: copy everything
        if (k >= 2) CU_TRY(cudaStreamWaitEvent(c->bs_in, c->be_out[h], 0));   // half h is free again
        CU_TRY(copy_others(bnc, src, c->bs_in));
        CU_TRY(cudaEventRecord(c->be_in[h], c->bs_in));
        CU_TRY(cudaStreamWaitEvent(stream, c->be_in[h], 0));
        P.count = n;
        P.dtag = decision_tag(0, (int)d.algo, (int)d.proto, P.nch, dtype, op, n, 0, kPathBounce);
        st = launch_kernel(c, fn, P, grid, stream, smem);
        if (st != POLAR_OK) return st;
        CU_TRY(cudaEventRecord(c->be_k[h], stream));
        CU_TRY(cudaStreamWaitEvent(c->bs_out, c->be_k[h], 0));
        CU_TRY(copy_others(src, bnc, c->bs_out));
        CU_TRY(cudaEventRecord(c->be_out[h], c->bs_out));
    }
    CU_TRY(cudaStreamWaitEvent(stream, c->be_out[(k - 1) & 1], 0));   // bs_out is in order: the last covers all
    return POLAR_OK;
}

// ReduceScatter (mode 0) / AllGather (1) / Broadcast (2): SURVEY f4.  count =
// elements per block (RS recvcount, AG sendcount, BC count).  Real comms need
// the peer-accessed buffers registered (RS: send, AG: recv, BC: buf).
polar_status do_direct(polar_comm_s* c, int mode, void* const* sends, void* const* recvs, size_t count, int dtype,
                       int op, int root, cudaStream_t stream) {
    const int es = esize_of(dtype);
    if (!es || (mode == 0 && !op_ok(op))) return POLAR_EINVAL;
    if (mode == 2 && (root < 0 || root >= c->nranks)) return POLAR_EINVAL;
    if (count > 0 && (!sends || (mode != 2 && !recvs))) return POLAR_EINVAL;
    for (int l = 0; l < c->nlocal && count > 0; ++l) {
        if (!sends[l] || (reinterpret_cast<uintptr_t>(sends[l]) % es)) return POLAR_EINVAL;
        if (mode != 2 && (!recvs[l] || (reinterpret_cast<uintptr_t>(recvs[l]) % es))) return POLAR_EINVAL;
    }
    polar_status st = check_latched(c);
    if (st != POLAR_OK) return st;
    static const uint32_t kColl[3] = {POLAR_COLL_REDUCESCATTER, POLAR_COLL_ALLGATHER, POLAR_COLL_BROADCAST};
    const uint64_t bytes = (uint64_t)count * (uint64_t)es * (mode == 2 ? 1u : (uint64_t)c->nranks);
    polar_ctx ctx{kColl[mode], (uint32_t)c->nranks, bytes};
    polar_decision d;
    st = polar_decide(&ctx, &d);
    if (st != POLAR_OK) return st;
    if (d.algo != POLAR_ALGO_ONESHOT || d.proto != POLAR_PROTO_SIMPLE) return POLAR_EUNSUPPORTED;
    c->last = d;
    if (c->is_virtual) {
        const int maxch = std::max(1, c->max_coop_blocks / c->nranks);
        if ((int)d.nchannels > maxch) d.nchannels = (uint32_t)maxch;
    } else if (c->share_cap > 0 && (int)d.nchannels > c->share_cap) {
        d.nchannels = (uint32_t)c->share_cap;
    }
    c->last_nch = d.nchannels;
    c->last_transport = POLAR_TRANSPORT_PEER;
    if (count == 0) return POLAR_OK;
    DeviceGuard dg(c->device);
    if (!dg.ok) return POLAR_ECUDA;
    const size_t blk = count * (size_t)es;
    if (c->nranks == 1) {   // identity collectives: copy send -> recv where they differ
        if (mode != 2 && sends[0] != recvs[0])
            CU_TRY(cudaMemcpyAsync(recvs[0], sends[0], blk, cudaMemcpyDeviceToDevice, stream));
        return POLAR_OK;
    }
    const void* fn = direct_kernel_for(dtype, mode, op);
    if (!fn) return POLAR_EUNSUPPORTED;
    dev::Params P;
    fill_params(c, P);
    P.nch = (int)d.nchannels;
    P.count = count;
    P.root = root;
    P.dtag = decision_tag(1 + mode, (int)d.algo, (int)d.proto, P.nch, dtype, op, count, root);
    const int grid = c->nlocal * P.nch;
    bool vec = mode == 2 || (blk % 16) == 0;
    auto aligned = [](const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; };
    if (c->is_virtual) {
        for (int p = 0; p < c->nranks; ++p) {
            P.bufs[p] = reinterpret_cast<char*>(sends[p]);
            P.recv[p] = mode == 2 ? nullptr : reinterpret_cast<char*>(recvs[p]);
            vec = vec && aligned(P.bufs[p]) && (mode == 2 || aligned(P.recv[p]));
        }
    } else {
        char* mine_s = reinterpret_cast<char*>(sends[0]);
        char* mine_r = mode == 2 ? nullptr : reinterpret_cast<char*>(recvs[0]);
        // the buffer peers access must be registered (symmetric), at the same offset on every rank
        char* shared = mode == 1 ? mine_r : mine_s;
        const size_t ext = mode == 2 ? blk : blk * (size_t)c->nranks;
        const Registration* reg = find_reg(c, shared, ext);
        if (!reg) return POLAR_EINVAL;
        const size_t off = (size_t)(shared - reg->base);
        P.dtag = decision_tag(1 + mode, (int)d.algo, (int)d.proto, P.nch, dtype, op, count, root,
                              ((uint64_t)(reg->id + 1) << 40) ^ (uint64_t)off);
        for (int p = 0; p < c->nranks; ++p) {
            char* peer = reg->peer[p] + off;
            if (mode == 1) {
                P.recv[p] = peer;
            } else {
                P.bufs[p] = peer;
            }
            vec = vec && aligned(peer);
        }
        if (mode == 0) P.recv[c->rank0] = mine_r;
        if (mode == 1) P.bufs[c->rank0] = mine_s;
        vec = vec && aligned(mine_s) && (mode == 2 || aligned(mine_r));
    }
    P.vec = vec;
    return launch_kernel(c, fn, P, grid, stream);
}

}  // namespace

extern "C" {

polar_status polar_comm_init(polar_comm_t* out, int nranks, int rank, int cuda_device, polar_allgather_fn ag,
                             void* user) {
    if (!out || nranks < 1 || nranks > POLAR_MAXRANKS || rank < 0 || rank >= nranks || !ag) return POLAR_EINVAL;
    *out = nullptr;
    polar_comm_s* c = new (std::nothrow) polar_comm_s;
    if (!c) return POLAR_ENOMEM;
    c->nranks = nranks;
    c->rank0 = rank;
    c->nlocal = 1;
    c->device = cuda_device;
    c->ag = ag;
    c->user = user;
    c->L = make_layout(true);
    {
        const char* e = std::getenv("POLAR_LL128_REAL");
        c->ll128_ok = e && e[0] == '1';
    }
    DeviceGuard dg(cuda_device);
    polar_status st = dg.ok ? POLAR_OK : POLAR_ECUDA;
    if (st == POLAR_OK) st = alloc_common(c);
    if (st == POLAR_OK) st = cuerr(cudaMalloc(reinterpret_cast<void**>(&c->scratch_own[0]), c->L.total));
    if (st == POLAR_OK) st = cuerr(cudaMemset(c->scratch_own[0], 0, c->L.total));
    if (st == POLAR_OK) st = cuerr(cudaDeviceSynchronize());
    cudaDeviceProp prop{};
    if (st == POLAR_OK) st = cuerr(cudaGetDeviceProperties(&prop, cuda_device));
    bool shared_gpu = false;
    int per_gpu = 1;
    if (st == POLAR_OK)
        st = bootstrap_check(nranks, rank, c->L, ag, user, reinterpret_cast<const unsigned char*>(prop.uuid.bytes),
                             &shared_gpu, &per_gpu);
    // Ranks sharing one GPU (MPS): every rank's CTAs must be resident together
    // or the cross-rank waits cannot complete, so the channel count is capped at
    // the co-resident CTAs / the ranks per GPU (the same cap on every rank: the
    // minimum over ranks); one rank per GPU (a node) has no cap.
    if (st == POLAR_OK && per_gpu > 1) {
        int blocks = 0;
        st = coresident_blocks(cuda_device, &blocks);
        uint32_t mine = (uint32_t)std::max(1, blocks / per_gpu), all[kMaxRanks];
        if (st == POLAR_OK && ag(&mine, all, sizeof(mine), user) != 0) st = POLAR_ESTATE;
        if (st == POLAR_OK) {
            for (int p = 0; p < nranks; ++p) mine = std::min(mine, all[p]);
            c->share_cap = (int)mine;
        }
    }
    // Ranks sharing one GPU (MPS) must not use programmatic dependent launch: a
    // rank's pre-launched next kernels can hold the SMs another rank's CURRENT
    // kernel needs, and the cross-rank waits then never complete (measured: 4
    // processes under MPS time out with PDL, run without).  One rank per GPU is
    // safe: a rank's own current kernel is always fully resident first.
    if (shared_gpu) c->pdl = false;
    if (st == POLAR_OK) st = exchange_and_map(c, c->scratch_own[0], c->scratch);
    if (st == POLAR_OK && nranks > 1 && c->L.nvls_bytes)
        st = nvls_setup(c->nvls, nranks, rank, cuda_device, ag, user, c->L.nvls_bytes);
    else if (st == POLAR_OK)
        std::snprintf(c->nvls.why, sizeof(c->nvls.why), "%s", nranks > 1 ? "disabled (POLAR_NVLS=0)" : "one rank");
    if (st == POLAR_OK) st = init_barrier(c);
    if (st != POLAR_OK) { destroy_comm(c, false); return st; }
    *out = c;
    return POLAR_OK;
}

polar_status polar_bootstrap_check(int nranks, int rank, polar_allgather_fn ag, void* user) {
    if (nranks < 1 || nranks > POLAR_MAXRANKS || rank < 0 || rank >= nranks || !ag) return POLAR_EINVAL;
    return bootstrap_check(nranks, rank, make_layout(true), ag, user);
}

polar_status polar_comm_init_virtual(polar_comm_t* out, int nranks, int cuda_device) {
    if (!out || nranks < 1 || nranks > POLAR_MAXRANKS) return POLAR_EINVAL;
    *out = nullptr;
    polar_comm_s* c = new (std::nothrow) polar_comm_s;
    if (!c) return POLAR_ENOMEM;
    c->nranks = nranks;
    c->rank0 = 0;
    c->nlocal = nranks;
    c->device = cuda_device;
    c->is_virtual = true;
    {
        // Plain launch + PDL by default, like real comms: the grid
        // is clamped to the co-resident bound, so every CTA becomes resident on an
        // otherwise idle GPU; the next call's CTAs are scheduled as this call's
        // drain (measured ~2 us per call less than a cooperative launch, whose
        // grid must wait for the whole previous grid to leave).  A foreign kernel
        // holding SMs can only delay residency into a bounded wait (ETIMEOUT),
        // not hang.  POLAR_VIRTUAL_COOP=1 forces cooperative launches.
        const char* ev = std::getenv("POLAR_VIRTUAL_COOP");
        c->coop = ev && ev[0] == '1';
    }
    c->L = make_layout(false);
    std::snprintf(c->nvls.why, sizeof(c->nvls.why),
                  "virtual comm: every rank on one device (a multicast object binds one region per device)");
    DeviceGuard dg(cuda_device);
    polar_status st = dg.ok ? POLAR_OK : POLAR_ECUDA;
    if (st == POLAR_OK) st = alloc_common(c);
    for (int p = 0; p < nranks && st == POLAR_OK; ++p) {
        st = cuerr(cudaMalloc(reinterpret_cast<void**>(&c->scratch_own[p]), c->L.total));
        if (st == POLAR_OK) st = cuerr(cudaMemset(c->scratch_own[p], 0, c->L.total));
        c->scratch[p] = c->scratch_own[p];
    }
    if (st == POLAR_OK) {
        st = coresident_blocks(cuda_device, &c->max_coop_blocks);
        if (st == POLAR_OK && c->max_coop_blocks < nranks) st = POLAR_EUNSUPPORTED;
    }
    if (st == POLAR_OK && nranks > 1) {
        const char* ec = std::getenv("POLAR_CLUSTER");
        c->cluster = !(ec && ec[0] == '0');
        // The cluster tree (down phase through L2) is faster than the FIFO tree at
        // every size measured (DESIGN.md §8 "Cluster transport"); the bound stays
        // as a knob (POLAR_CLUSTER_TREE_MAX bytes per rank, default: none)
        c->cl_tree_max = env_size("POLAR_CLUSTER_TREE_MAX", ~(size_t)0);
        for (int algo : {POLAR_ALGO_RING, POLAR_ALGO_TREE})
            c->cl_max_ch[algo] = c->cluster ? std::min(POLAR_MAXCH, cluster_max_active(algo, nranks)) : 0;
    }
    if (st == POLAR_OK) st = cuerr(cudaDeviceSynchronize());
    if (st == POLAR_OK) st = init_barrier(c);
    if (st != POLAR_OK) { destroy_comm(c, false); return st; }
    *out = c;
    return POLAR_OK;
}

polar_status polar_comm_destroy(polar_comm_t comm) {
    if (!comm) return POLAR_EINVAL;
    destroy_comm(comm, true);
    return POLAR_OK;
}

polar_status polar_comm_info(polar_comm_t comm, int* nranks, int* rank, int* nlocal) {
    if (!comm) return POLAR_EINVAL;
    if (nranks) *nranks = comm->nranks;
    if (rank) *rank = comm->rank0;
    if (nlocal) *nlocal = comm->nlocal;
    return POLAR_OK;
}

polar_status polar_mem_alloc(polar_comm_t comm, size_t bytes, void** ptrs) {
    if (!comm || !ptrs || bytes == 0) return POLAR_EINVAL;
    std::lock_guard<std::mutex> lk(comm->mu);
    DeviceGuard dg(comm->device);
    if (!dg.ok) return POLAR_ECUDA;
    if (comm->is_virtual) {
        for (int p = 0; p < comm->nranks; ++p) {
            char* m = nullptr;
            if (cudaMalloc(reinterpret_cast<void**>(&m), bytes) != cudaSuccess) return POLAR_ENOMEM;
            comm->virt_allocs.push_back(m);
            ptrs[p] = m;
        }
        return POLAR_OK;
    }
    Registration r{};
    if (cudaMalloc(reinterpret_cast<void**>(&r.base), bytes) != cudaSuccess) return POLAR_ENOMEM;
    r.bytes = bytes;
    r.owned = true;
    r.id = comm->reg_seq++;
    r.buffer_id = buffer_id_of(r.base);
    polar_status st = exchange_and_map(comm, r.base, r.peer, r.peer_base);
    if (st != POLAR_OK) { cudaFree(r.base); return st; }
    comm->regs.push_back(r);
    ptrs[0] = r.base;
    return POLAR_OK;
}

polar_status polar_mem_free(polar_comm_t comm, void* ptr) {
    if (!comm || !ptr) return POLAR_EINVAL;
    std::lock_guard<std::mutex> lk(comm->mu);
    DeviceGuard dg(comm->device);
    cudaDeviceSynchronize();
    for (size_t i = 0; i < comm->virt_allocs.size(); ++i)
        if (comm->virt_allocs[i] == ptr) {
            cudaFree(ptr);
            comm->virt_allocs.erase(comm->virt_allocs.begin() + (long)i);
            return POLAR_OK;
        }
    for (size_t i = 0; i < comm->regs.size(); ++i)
        if (comm->regs[i].base == ptr && comm->regs[i].owned) {
            // collective: everyone is done with every copy, everyone unmaps the
            // peers' copies (each owned buffer is its own allocation, mapped at
            // offset 0), everyone has unmapped, then each rank frees its own
            polar_status st = host_barrier(comm);
            release_registration(comm, i);
            if (st == POLAR_OK) st = host_barrier(comm);
            cudaFree(ptr);
            return st;
        }
    return POLAR_EINVAL;
}

polar_status polar_register(polar_comm_t comm, void* buf, size_t bytes) {
    if (!comm || !buf || bytes == 0) return POLAR_EINVAL;
    if (comm->is_virtual) return POLAR_OK;
    std::lock_guard<std::mutex> lk(comm->mu);
    DeviceGuard dg(comm->device);
    if (!dg.ok) return POLAR_ECUDA;
    Registration r{};
    r.base = reinterpret_cast<char*>(buf);
    r.bytes = bytes;
    r.owned = false;
    r.id = comm->reg_seq++;
    r.buffer_id = buffer_id_of(buf);
    polar_status st = exchange_and_map(comm, r.base, r.peer, r.peer_base);
    if (st != POLAR_OK) return st;
    comm->regs.push_back(r);
    return POLAR_OK;
}

polar_status polar_deregister(polar_comm_t comm, void* buf) {
    if (!comm || !buf) return POLAR_EINVAL;
    if (comm->is_virtual) return POLAR_OK;
    std::lock_guard<std::mutex> lk(comm->mu);
    DeviceGuard dg(comm->device);
    if (!dg.ok) return POLAR_ECUDA;
    cudaDeviceSynchronize();
    polar_status st = host_barrier(comm);   // no peer still reads or writes through the mappings
    for (size_t i = 0; i < comm->regs.size(); ++i)
        if (comm->regs[i].base == buf && !comm->regs[i].owned) {
            release_registration(comm, i);
            break;
        }
    // (not registered here, or already dropped as stale: still collective, still OK)
    return st;
}

polar_status polar_comm_autoreg(polar_comm_t comm, int enable, size_t min_bytes) {
    if (!comm) return POLAR_EINVAL;
    const size_t want = enable ? min_bytes : ~(size_t)0;
    std::lock_guard<std::mutex> lk(comm->mu);
    if (!comm->is_virtual && comm->nranks > 1) {
        // collective: every rank must exchange on the same calls
        if (!comm->ag) return POLAR_EINVAL;
        unsigned long long mine = want, all[kMaxRanks];
        if (comm->ag(&mine, all, sizeof(mine), comm->user) != 0) return POLAR_ESTATE;
        for (int p = 0; p < comm->nranks; ++p)
            if (all[p] != mine) return POLAR_EINVAL;
    }
    comm->autoreg_min = want;
    return POLAR_OK;
}

polar_status polar_comm_autoreg_stats(polar_comm_t comm, polar_autoreg_stats* out) {
    if (!comm || !out) return POLAR_EINVAL;
    std::lock_guard<std::mutex> lk(comm->mu);
    *out = comm->ar;
    return POLAR_OK;
}

polar_status polar_allreduce(polar_comm_t comm, void* buf, size_t count, polar_dtype dtype, polar_op op,
                             void* stream) {
    if (!comm) return POLAR_EINVAL;
    if (comm->nlocal != 1) return POLAR_EINVAL;
    void* bufs[1] = {buf};
    return do_allreduce(comm, bufs, count, dtype, op, nullptr, reinterpret_cast<cudaStream_t>(stream));
}

polar_status polar_allreduce_v(polar_comm_t comm, void* const* bufs, size_t count, polar_dtype dtype, polar_op op,
                               void* stream) {
    if (!comm) return POLAR_EINVAL;
    return do_allreduce(comm, bufs, count, dtype, op, nullptr, reinterpret_cast<cudaStream_t>(stream));
}

polar_status polar_allreduce_forced(polar_comm_t comm, void* const* bufs, size_t count, polar_dtype dtype,
                                    polar_op op, const polar_decision* forced, void* stream) {
    if (!comm || !forced) return POLAR_EINVAL;
    return do_allreduce(comm, bufs, count, dtype, op, forced, reinterpret_cast<cudaStream_t>(stream));
}

polar_status polar_reduce_scatter(polar_comm_t comm, const void* sendbuf, void* recvbuf, size_t recvcount,
                                  polar_dtype dtype, polar_op op, void* stream) {
    if (!comm || comm->nlocal != 1) return POLAR_EINVAL;
    void* s[1] = {const_cast<void*>(sendbuf)};
    void* r[1] = {recvbuf};
    return do_direct(comm, 0, s, r, recvcount, dtype, op, 0, reinterpret_cast<cudaStream_t>(stream));
}

polar_status polar_reduce_scatter_v(polar_comm_t comm, void* const* sendbufs, void* const* recvbufs, size_t recvcount,
                                    polar_dtype dtype, polar_op op, void* stream) {
    if (!comm) return POLAR_EINVAL;
    return do_direct(comm, 0, sendbufs, recvbufs, recvcount, dtype, op, 0, reinterpret_cast<cudaStream_t>(stream));
}

polar_status polar_all_gather(polar_comm_t comm, const void* sendbuf, void* recvbuf, size_t sendcount,
                              polar_dtype dtype, void* stream) {
    if (!comm || comm->nlocal != 1) return POLAR_EINVAL;
    void* s[1] = {const_cast<void*>(sendbuf)};
    void* r[1] = {recvbuf};
    return do_direct(comm, 1, s, r, sendcount, dtype, POLAR_SUM, 0, reinterpret_cast<cudaStream_t>(stream));
}

polar_status polar_all_gather_v(polar_comm_t comm, void* const* sendbufs, void* const* recvbufs, size_t sendcount,
                                polar_dtype dtype, void* stream) {
    if (!comm) return POLAR_EINVAL;
    return do_direct(comm, 1, sendbufs, recvbufs, sendcount, dtype, POLAR_SUM, 0, reinterpret_cast<cudaStream_t>(stream));
}

polar_status polar_broadcast(polar_comm_t comm, void* buf, size_t count, polar_dtype dtype, int root, void* stream) {
    if (!comm || comm->nlocal != 1) return POLAR_EINVAL;
    void* b[1] = {buf};
    return do_direct(comm, 2, b, nullptr, count, dtype, POLAR_SUM, root, reinterpret_cast<cudaStream_t>(stream));
}

polar_status polar_broadcast_v(polar_comm_t comm, void* const* bufs, size_t count, polar_dtype dtype, int root,
                               void* stream) {
    if (!comm) return POLAR_EINVAL;
    return do_direct(comm, 2, bufs, nullptr, count, dtype, POLAR_SUM, root, reinterpret_cast<cudaStream_t>(stream));
}

polar_status polar_allreduce_host(polar_comm_t comm, void* const* host_bufs, void* const* dev_bufs, size_t count,
                                  polar_dtype dtype, polar_op op, void* stream) {
    if (!comm || (count && (!host_bufs || !dev_bufs))) return POLAR_EINVAL;
    const int es = esize_of(dtype);
    if (!es) return POLAR_EINVAL;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    DeviceGuard dg(comm->device);
    if (!dg.ok) return POLAR_ECUDA;
    if (count == 0) return do_allreduce(comm, dev_bufs, 0, dtype, op, nullptr, s);
    // Chunk pipeline: H2D of chunk k+1 (copy stream in), the AllReduce of chunk k
    // (the caller's stream) and D2H of chunk k-1 (copy stream out) overlap, so the
    // two PCIe directions run concurrently.  Each chunk is an independent
    // AllReduce of a contiguous element range (decided by its own bytes); the
    // result is the AllReduce of the whole message because the op is elementwise.
    if (!comm->hs_in) {
        CU_TRY(cudaStreamCreateWithFlags(&comm->hs_in, cudaStreamNonBlocking));
        CU_TRY(cudaStreamCreateWithFlags(&comm->hs_out, cudaStreamNonBlocking));
        CU_TRY(cudaEventCreateWithFlags(&comm->he_start, cudaEventDisableTiming));
        CU_TRY(cudaEventCreateWithFlags(&comm->he_in, cudaEventDisableTiming));
        CU_TRY(cudaEventCreateWithFlags(&comm->he_red, cudaEventDisableTiming));
        CU_TRY(cudaEventCreateWithFlags(&comm->he_out, cudaEventDisableTiming));
    }
    const size_t chunk_bytes = env_size("POLAR_HOST_CHUNK", 8u << 20);
    size_t chunk = std::max<size_t>(1, chunk_bytes / (size_t)es);
    chunk = std::max<size_t>(16 / es, chunk / (16 / es) * (16 / es));   // keep chunk starts 16-B aligned
    CU_TRY(cudaEventRecord(comm->he_start, s));
    CU_TRY(cudaStreamWaitEvent(comm->hs_in, comm->he_start, 0));
    CU_TRY(cudaStreamWaitEvent(comm->hs_out, comm->he_start, 0));
    std::vector<void*> sub(comm->nlocal);
    for (size_t done = 0; done < count; done += chunk) {
        const size_t n = std::min(chunk, count - done);
        const size_t off = done * (size_t)es, nb = n * (size_t)es;
        for (int l = 0; l < comm->nlocal; ++l)
            CU_TRY(cudaMemcpyAsync(static_cast<char*>(dev_bufs[l]) + off, static_cast<const char*>(host_bufs[l]) + off,
                                   nb, cudaMemcpyHostToDevice, comm->hs_in));
        CU_TRY(cudaEventRecord(comm->he_in, comm->hs_in));
        CU_TRY(cudaStreamWaitEvent(s, comm->he_in, 0));
        for (int l = 0; l < comm->nlocal; ++l) sub[l] = static_cast<char*>(dev_bufs[l]) + off;
        polar_status st = do_allreduce(comm, sub.data(), n, dtype, op, nullptr, s);
        if (st != POLAR_OK) {
            cudaStreamSynchronize(comm->hs_in);
            cudaStreamSynchronize(comm->hs_out);
            return st;
        }
        CU_TRY(cudaEventRecord(comm->he_red, s));
        CU_TRY(cudaStreamWaitEvent(comm->hs_out, comm->he_red, 0));
        for (int l = 0; l < comm->nlocal; ++l)
            CU_TRY(cudaMemcpyAsync(static_cast<char*>(host_bufs[l]) + off, static_cast<char*>(dev_bufs[l]) + off, nb,
                                   cudaMemcpyDeviceToHost, comm->hs_out));
    }
    CU_TRY(cudaEventRecord(comm->he_out, comm->hs_out));
    CU_TRY(cudaStreamWaitEvent(s, comm->he_out, 0));
    CU_TRY(cudaStreamSynchronize(s));
    return check_latched(comm);
}

polar_status polar_comm_probe_ll128(polar_comm_t comm, unsigned long long iters, unsigned long long* torn_lanes,
                                   unsigned long long* lane_reads) {
    if (!comm || iters < 1 || !torn_lanes || !lane_reads) return POLAR_EINVAL;
    polar_status st = check_latched(comm);
    if (st != POLAR_OK) return st;
    if (comm->is_virtual || comm->nranks == 1) {
        // one device: the single-GPU probe is the transport's probe
        st = polar_probe_ll128(comm->device, kProbePairs, iters, 0, 0, torn_lanes, lane_reads);
        if (st == POLAR_OK) comm->ll128_ok = *torn_lanes == 0 && *lane_reads > 0;
        return st;
    }
    DeviceGuard dg(comm->device);
    if (!dg.ok) return POLAR_ECUDA;
    const int r = comm->rank0, n = comm->nranks, next = (r + 1) % n, prev = (r + n - 1) % n;
    const size_t fifo_bytes = (size_t)kProbePairs * 8 * 512;
    char* mine = comm->scratch[r] + comm->L.probe_off;
    unsigned long long* cnt = nullptr;
    CU_TRY(cudaDeviceSynchronize());
    if (cudaMalloc(&cnt, 16) != cudaSuccess) return POLAR_ENOMEM;
    st = cuerr(cudaMemset(mine, 0, probe_ll128_region_bytes(kProbePairs)));
    if (st == POLAR_OK) st = cuerr(cudaMemset(cnt, 0, 16));
    if (st == POLAR_OK) st = cuerr(cudaDeviceSynchronize());
    if (st == POLAR_OK) st = host_barrier(comm);   // every region zeroed before anyone writes
    if (st == POLAR_OK) {
        char* to = comm->scratch[next] + comm->L.probe_off;
        char* from = comm->scratch[prev] + comm->L.probe_off;
        st = cuerr(launch_probe_ll128_xrank(reinterpret_cast<uint4*>(to),
                                            reinterpret_cast<unsigned long long*>(mine + fifo_bytes),
                                            reinterpret_cast<uint4*>(mine),
                                            reinterpret_cast<unsigned long long*>(from + fifo_bytes), kProbePairs,
                                            iters, cnt, comm->timeout_ns, comm->err_dev));
    }
    if (st == POLAR_OK) st = cuerr(cudaDeviceSynchronize());
    unsigned long long h[2] = {0, 0};
    if (st == POLAR_OK) st = cuerr(cudaMemcpy(h, cnt, 16, cudaMemcpyDeviceToHost));
    cudaFree(cnt);
    if (st == POLAR_OK) st = check_latched(comm);
    // every rank learns every rank's count: the gate opens on all ranks or none
    struct Rec { unsigned long long torn, reads; int32_t st, pad; } me{h[0], h[1], (int32_t)st, 0};
    std::vector<Rec> all(n);
    if (comm->ag(&me, all.data(), sizeof(Rec), comm->user) != 0) return POLAR_ESTATE;
    unsigned long long torn = 0, reads = 0;
    bool ok = true;
    for (const Rec& x : all) {
        torn += x.torn;
        reads += x.reads;
        ok = ok && x.st == POLAR_OK;
    }
    *torn_lanes = torn;
    *lane_reads = reads;
    comm->ll128_ok = ok && torn == 0 && reads == (unsigned long long)n * kProbePairs * iters * 32;
    return st != POLAR_OK ? st : (ok ? POLAR_OK : POLAR_ESTATE);
}

polar_status polar_comm_nvls_info(polar_comm_t comm, int* available, char* why, size_t len) {
    if (!comm) return POLAR_EINVAL;
    if (available) *available = comm->nvls.ok ? 1 : 0;
    if (why && len) std::snprintf(why, len, "%s", comm->nvls.why);
    return POLAR_OK;
}

polar_status polar_comm_last_decision(polar_comm_t comm, polar_decision* out) {
    if (!comm || !out) return POLAR_EINVAL;
    *out = comm->last;
    return POLAR_OK;
}

polar_status polar_comm_launch_info(polar_comm_t comm, uint32_t* nchannels, uint32_t* grid) {
    if (!comm) return POLAR_EINVAL;
    if (nchannels) *nchannels = comm->last_nch;
    if (grid) *grid = comm->last_nch * (uint32_t)comm->nlocal;
    return POLAR_OK;
}

polar_status polar_comm_transport(polar_comm_t comm, int* transport) {
    if (!comm || !transport) return POLAR_EINVAL;
    *transport = comm->last_transport;
    return POLAR_OK;
}

uint64_t polar_comm_launches(polar_comm_t comm) { return comm ? comm->launches : 0; }

polar_status polar_comm_check(polar_comm_t comm) {
    if (!comm) return POLAR_EINVAL;
    return check_latched(comm);
}

polar_status polar_comm_set_trace(polar_comm_t comm, void* dev_buf, size_t bytes) {
    if (!comm || (dev_buf && bytes < (size_t)comm->nlocal * POLAR_MAXCH * 4 * sizeof(unsigned long long)))
        return POLAR_EINVAL;
    comm->trace = reinterpret_cast<unsigned long long*>(dev_buf);
    return POLAR_OK;
}

polar_status polar_bench_enqueue(polar_comm_t comm, void* const* bufs, size_t count, polar_dtype dtype,
                                 polar_op op, void* stream, uint64_t ncalls, double* ns_per_call) {
    if (!comm || !ns_per_call || ncalls == 0) return POLAR_EINVAL;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    polar_status st = do_allreduce(comm, bufs, count, dtype, op, nullptr, s);   // warm
    if (st != POLAR_OK) return st;
    CU_TRY(cudaStreamSynchronize(s));
    auto t0 = std::chrono::steady_clock::now();
    for (uint64_t i = 0; i < ncalls; ++i) {
        st = do_allreduce(comm, bufs, count, dtype, op, nullptr, s);
        if (st != POLAR_OK) return st;
    }
    auto t1 = std::chrono::steady_clock::now();
    CU_TRY(cudaStreamSynchronize(s));
    *ns_per_call = std::chrono::duration<double, std::nano>(t1 - t0).count() / (double)ncalls;
    return check_latched(comm);
}

polar_status polar_adaptive_config(polar_comm_t comm, const polar_adaptive_params* params) {
    if (!comm || !params) return POLAR_EINVAL;
    polar_status st = adaptive_validate(*params);
    if (st != POLAR_OK) return st;
    adaptive_reset(comm->ad, *params);
    comm->tel_consumed = comm->tel_seq;   // forget samples of earlier calls
    return POLAR_OK;
}

polar_status polar_adaptive_inject(polar_comm_t comm, double latency_scale) {
    if (!comm || !(latency_scale > 0.0)) return POLAR_EINVAL;
    comm->ad.prm.latency_scale = latency_scale;
    return POLAR_OK;
}

polar_status polar_adaptive_get_state(polar_comm_t comm, polar_adaptive_state* out) {
    if (!comm || !out) return POLAR_EINVAL;
    adaptive_drain(comm);
    out->channels = comm->ad.c;
    out->contended = comm->ad.contended ? 1u : 0u;
    out->windows = comm->ad.windows;
    out->samples = comm->ad.samples;
    out->last_mean_ns = comm->ad.last_mean;
    return POLAR_OK;
}

polar_status polar_p2p_probe(polar_comm_t comm, void* const* bufs, size_t bytes, int iters, polar_p2p_result* out) {
    if (!comm || !bufs || !out || bytes < 16 || bytes % 16 || iters < 1) return POLAR_EINVAL;
    polar_status st = check_latched(comm);
    if (st != POLAR_OK) return st;
    DeviceGuard dg(comm->device);
    if (!dg.ok) return POLAR_ECUDA;
    dev::Params P;
    fill_params(comm, P);
    int nch = POLAR_MAXCH;
    if (comm->is_virtual) nch = std::max(1, std::min(nch, comm->max_coop_blocks / comm->nranks));
    P.nch = nch;
    P.count = bytes;
    P.vec = 1;
    if (comm->is_virtual) {
        for (int p = 0; p < comm->nranks; ++p) {
            if (!bufs[p] || reinterpret_cast<uintptr_t>(bufs[p]) % 16) return POLAR_EINVAL;
            P.bufs[p] = static_cast<char*>(bufs[p]);
        }
    } else {
        const Registration* reg = find_reg(comm, static_cast<const char*>(bufs[0]), bytes);
        if (!reg || reinterpret_cast<uintptr_t>(bufs[0]) % 16) return POLAR_EINVAL;
        const size_t off = (size_t)(static_cast<const char*>(bufs[0]) - reg->base);
        for (int p = 0; p < comm->nranks; ++p) P.bufs[p] = reg->peer[p] + off;
    }
    const int grid = comm->nlocal * nch;
    unsigned long long *times = nullptr, *sums = nullptr;
    if (cudaMalloc(&times, sizeof(unsigned long long) * 2 * grid) != cudaSuccess) return POLAR_ENOMEM;
    if (cudaMalloc(&sums, sizeof(unsigned long long) * grid) != cudaSuccess) { cudaFree(times); return POLAR_ENOMEM; }
    std::vector<unsigned long long> ht(2 * grid);
    for (int l = 0; l < comm->nlocal; ++l) out[l] = polar_p2p_result{};
    for (int mode = dev::PROBE_LOAD; mode <= dev::PROBE_PINGPONG && st == POLAR_OK; ++mode) {
        unsigned long long epoch = ++comm->probe_epoch;
        void* args[] = {&P, &mode, &iters, &epoch, &times, &sums};
        cudaError_t e = comm->is_virtual
                            ? cudaLaunchCooperativeKernel((const void*)dev::p2p_probe_kernel, dim3(grid), dim3(dev::kBlock), args, 0, 0)
                            : cudaLaunchKernel((const void*)dev::p2p_probe_kernel, dim3(grid), dim3(dev::kBlock), args, 0, 0);
        if (e != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) { st = POLAR_ECUDA; break; }
        comm->launches++;
        st = check_latched(comm);
        if (st != POLAR_OK) break;
        if (cudaMemcpy(ht.data(), times, sizeof(unsigned long long) * 2 * grid, cudaMemcpyDeviceToHost) != cudaSuccess) {
            st = POLAR_ECUDA;
            break;
        }
        for (int l = 0; l < comm->nlocal; ++l) {
            unsigned long long t0 = ~0ull, t1 = 0;
            for (int ch = 0; ch < nch; ++ch) {
                t0 = std::min(t0, ht[2 * (l * nch + ch)]);
                t1 = std::max(t1, ht[2 * (l * nch + ch) + 1]);
            }
            const double ns = (double)(t1 - t0);
            if (mode == dev::PROBE_LOAD) out[l].load_gbs = ns > 0 ? (double)bytes * iters / ns : 0.0;
            if (mode == dev::PROBE_STORE) out[l].store_gbs = ns > 0 ? (double)bytes * iters / ns : 0.0;
            if (mode == dev::PROBE_PINGPONG) {
                const int r = comm->rank0 + l;
                const double pp = (double)(ht[2 * (l * nch) + 1] - ht[2 * (l * nch)]);
                out[l].pingpong_us = (r ^ 1) < comm->nranks ? pp / iters / 1e3 : 0.0;
            }
        }
        if (mode == dev::PROBE_LOAD) {
            std::vector<unsigned long long> hs(grid);
            cudaMemcpy(hs.data(), sums, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost);
            for (int l = 0; l < comm->nlocal; ++l) {
                unsigned long long x = 0;
                for (int ch = 0; ch < nch; ++ch) x ^= hs[l * nch + ch];
                out[l].load_xor = x;
            }
        }
    }
    cudaFree(times);
    cudaFree(sums);
    return st;
}

const char* polar_version(void) { return "polar 0.1 sm_100a"; }

}  // extern "C"
