// Device primitives for the polar kernels (sm_100a): cross-rank flags, LL lines,
// 16-byte packs with partial tails, and the reduction arithmetic (SURVEY.md §8(a)
// rows a7, a8, a10, a11).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "polar.h"
#include "polar_internal.h"

namespace polar {
namespace dev {

// ------------------------------------------------------------- kernel params

#ifndef POLAR_BLOCK
#define POLAR_BLOCK 512
#endif
#ifndef POLAR_LB_MIN
#define POLAR_LB_MIN 1      // min resident CTAs per SM requested from ptxas (register cap; 2 spills)
#endif
constexpr int kBlock = POLAR_BLOCK;   // threads per CTA (one CTA per rank-channel)

struct Params {
    char* bufs[kMaxRanks];     // rank p's data for this call (peer-mapped; zero-copy two-shot uses all)
    char* scratch[kMaxRanks];  // rank p's scratch base (peer-mapped)
    unsigned long long count;  // elements
    int nranks;                // ranks in the comm
    int rank0;                 // first rank hosted by this launch
    int nch;                   // channels (CTAs per rank)
    int vec;                   // 1: every buffer of this call is 16-B aligned
    int* err;                  // host-mapped error word (first error wins)
    unsigned long long timeout_ns;
    // layout (identical on every rank)
    unsigned long long flags_off, state_off;
    unsigned long long os_off, os_chunk, osll_off, osll_chunk, tsll_off, tsll_chunk;
    unsigned long long ring_off, ring_slot, ringll_off, ringll_slot;
    unsigned long long tree_off, tree_slot, treell_off, treell_slot;
    // LL128 regions (own memory: a stale line of another protocol must never be
    // read as LL128 and vice versa); staging slots are as large as the LL ones
    unsigned long long os128_off, ts128_off, ring128_off, ring128_slot, tree128_off, tree128_slot;
    unsigned long long* trace;  // optional per-CTA timestamps (polar_comm_set_trace), else null
    int sys;                    // 1: peers are other GPUs (system-scope ordering); 0: one GPU (gpu scope)
    int tma;                    // two-shot Simple: 1 = TMA bulk-copy staging through shared memory
    int ring_tma;               // ring Simple: 1 = TMA-staged FIFO kernel (ring_simple_tma) where eligible
    int ring_flags;             // ring_simple_tma: bit 0 = L2 eviction hints, bit 1 = discard consumed FIFO lines
    unsigned jitter_ns;         // fault injection: random __nanosleep (< jitter_ns) before 1/8 of all
                                // signal and LL stores (POLAR_JITTER_NS; 0 = off)
    TelEntry* tel;              // profiler telemetry ring (host-mapped), or null
    unsigned long long seq;     // this launch's sequence number in the ring
    // cross-rank decision check (real comms; kernels.cuh tag_begin / tag_end)
    unsigned long long tags_off;  // tag ring in every rank's scratch
    unsigned long long call;      // this launch's index on the comm (same on every rank)
    unsigned long long dtag;      // this launch's decision tag
    unsigned long long prev_tag;  // the previous launch's tag (call - 1)
    // direct collectives (ReduceScatter / AllGather / Broadcast)
    char* recv[kMaxRanks];      // rank p's receive buffer (RS / AG), peer-mapped
    int root;                   // Broadcast root
};


// -------------------------------------------------------------- raw memory ops

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Diagnostic: CTA b records %globaltimer at point k (0..3) into trace[4b+k].
__device__ __forceinline__ void trace_point(const Params& P, int k) {
    if (P.trace && threadIdx.x == 0) P.trace[4 * blockIdx.x + k] = globaltimer();
}

// Flag operations at system scope (peers on other GPUs over NVLink) or gpu scope
// (virtual ranks: every peer is on this GPU, so gpu-scope ordering suffices and
// avoids MEMBAR.SYS).  `sys` is uniform per launch.
__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v, int sys) {
    if (sys) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    else asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v, int sys) {
    if (sys) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    else asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p, int sys) {
    uint64_t v;
    if (sys) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel(int sys) {
    if (sys) asm volatile("fence.acq_rel.sys;" ::: "memory");
    else asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// data loads that must not hit a stale L1 line (peer data, staging reused within a kernel)
__device__ __forceinline__ uint4 ld_cg(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
// 16-B data store with an explicit global address space (STG.E.128; a plain
// `*p = v` through the char* scratch/peer tables compiles to a generic ST.E.128)
__device__ __forceinline__ void st_plain(uint4* p, uint4 v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// Consumed Simple staging / FIFO data: drop its L2 lines without write-back
// (`discard.global.L2`).  The bytes were written by a peer, read once, and will be
// overwritten before they are read again (the next lap of the FIFO / the next
// call), so writing the dirty lines back to HBM is wasted bandwidth.  The slot's
// contents become undefined, which Simple tolerates: a fill flag published after
// the next write, never the data itself, says when a slot is valid.  The whole
// CTA calls this after a barrier that ends every read of [p, p + bytes); p is
// 128-B aligned, and the last partial line is dropped too (its tail is unused).
// Off by default: measured on 8 virtual ranks (profiles/r01_discard_ab.jsonl) the
// ring's DRAM traffic falls to ~2.1 n S and 128 MiB runs 948 -> 887 us, but the
// extra barrier per step costs more everywhere else (ring 1 MiB 38.7 -> 42.0 us,
// tree 128 MiB 1269 -> 1346 us, one-shot 8 MiB 164 -> 177 us).
#ifndef POLAR_DISCARD
#define POLAR_DISCARD 0
#endif
__device__ __forceinline__ void discard_l2(const void* p, unsigned long long bytes) {
#if POLAR_DISCARD
    const char* c = static_cast<const char*>(p);
    for (unsigned long long o = (unsigned long long)threadIdx.x * 128; o < bytes; o += (unsigned long long)blockDim.x * 128)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(c + o) : "memory");
#endif
}

// LL line: 16 B = {d0, flag, d1, flag}; written with one 16-B volatile store,
// polled with one 16-B volatile load.
__device__ __forceinline__ void st_ll(uint4* p, uint32_t d0, uint32_t d1, uint32_t flag) {
    asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(d0), "r"(flag), "r"(d1),
                 "r"(flag)
                 : "memory");
}
__device__ __forceinline__ uint4 ld_ll(const uint4* p) {
    uint4 v;
    asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}

// LL128 (the protocol the paper's `nvlink_ring_mid_v2` policy
// selects for 4-32 MiB).  One warp moves a UNIT of 30 packs
// (480 B payload) as one group of 4 x 128-B lines (512 B on the wire, 93.75 %
// payload): in line g (lanes 8g..8g+7) lanes 8g..8g+6 carry packs 7g..7g+6 and
// lane 8g+7 carries 8 B of pack 28 + g/2 (low half for even g, high half for odd
// g) followed by the u64 flag in the line's last 8 B.  Each lane writes its 16 B
// with one st.volatile.v4; the warp's store of a 128-B line lands as one unit
// (the property NCCL's LL128 also relies on), so a reader that sees the flag of
// a line sees its data.  Readers load whole line groups and retry until all four
// flags match.  Warp-collective: every lane of the warp must call both.
constexpr int kLL128Packs = 30;
constexpr int kLL128UnitBytes = 512;

__device__ __forceinline__ void st_ll128(uint4* group, uint4 v, uint64_t flag) {
    const int lane = (int)(threadIdx.x & 31), g = lane >> 3, q = lane & 7;
    const int src = q < 7 ? g * 7 + q : 28 + (g >> 1);
    uint4 w;
    w.x = __shfl_sync(0xffffffffu, v.x, src);
    w.y = __shfl_sync(0xffffffffu, v.y, src);
    w.z = __shfl_sync(0xffffffffu, v.z, src);
    w.w = __shfl_sync(0xffffffffu, v.w, src);
    // flag lane: its half of pack 28 + g/2 in the low 8 B, the flag in the high 8 B
    // (selects, not branches: the store below must be issued by the whole warp)
    const bool fl = q == 7, hi = (g & 1) != 0;
    w.x = fl && hi ? w.z : w.x;
    w.y = fl && hi ? w.w : w.y;
    w.z = fl ? (uint32_t)flag : w.z;
    w.w = fl ? (uint32_t)(flag >> 32) : w.w;
    asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(group + lane), "r"(w.x), "r"(w.y), "r"(w.z),
                 "r"(w.w)
                 : "memory");
}

// ----------------------------------------------------- TMA bulk copies + mbarrier
constexpr int kTmaStages = 6;                           // 5 stages in flight while one is reduced
constexpr size_t kTmaStageBytes = 32 << 10;             // n tiles per stage, 32 KiB whatever n
__host__ __device__ constexpr unsigned tma_tile_packs(int n) { return (unsigned)(kTmaStageBytes / 16 / n); }
// dynamic shared memory of the TMA two-shot: stages + mbarriers + metadata
__host__ __device__ constexpr size_t tma_smem_bytes(int /*n*/) {
    return (size_t)kTmaStages * kTmaStageBytes + kTmaStages * (8 + 8 + 8 + 8) + 128;
}

// TMA-staged ring Simple (kernels.cuh ring_simple_tma): stages of one tile =
// the predecessor's FIFO words (sized for bf16's 2 f32 words per pack) + my packs
#ifndef POLAR_RING_TMA_STAGES
#define POLAR_RING_TMA_STAGES 6
#endif
#ifndef POLAR_RING_TMA_TILE
#define POLAR_RING_TMA_TILE 512
#endif
constexpr int kRtStages = POLAR_RING_TMA_STAGES;
constexpr unsigned kRtTile = POLAR_RING_TMA_TILE;       // element packs per tile (8 KiB of elements)
constexpr size_t kRtInBytes = (size_t)kRtTile * 16 * 2; // FIFO words of a tile, sized for AW = 2
constexpr size_t kRtStageBytes = kRtInBytes + (size_t)kRtTile * 16;
__host__ __device__ constexpr size_t ring_tma_smem_bytes() {
    return (size_t)kRtStages * kRtStageBytes + (size_t)kRtStages * 3 * 8 + 64;
}

// cp.async.bulk (SASS UBLKCP) moves whole tiles between global memory (local or
// peer-mapped) and shared memory; completion of loads is tracked by an mbarrier
// transaction count, stores by bulk async-groups.

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(smem_dst)),
                 "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* smem_src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(smem_src)),
                 "r"(bytes)
                 : "memory");
}
// L2 eviction-priority policies for bulk copies (createpolicy; SASS UBLKCP with a
// cache-policy operand): streaming data evict_first, FIFO lines that the
// consumer reads soon evict_last.
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_load_hint(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                               uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(smem_dst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void bulk_store_hint(void* gdst, const void* smem_src, uint32_t bytes, uint64_t pol) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
                 "r"(smem_u32(smem_src)), "r"(bytes), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N> __device__ __forceinline__ void bulk_wait_group() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// Fault injection: delay a random 1/8 of the signalling stores so
// that every protocol is exercised under skewed arrival orders.  jitter() draws
// per thread (LL lines and flags are per-thread stores); jitter_warp() draws
// once per warp, for LL128, whose premise is a CONVERGENT warp store: per-lane
// NANOSLEEP delays right before the store were measured to split it and tear
// lines (polar_probe_ll128, profiles/r01_probe_ll128.jsonl).
__device__ __forceinline__ void jitter(const Params& P) {
    if (P.jitter_ns == 0) return;
    uint32_t x = (uint32_t)globaltimer() * 2654435761u ^ (threadIdx.x * 40503u) ^ (blockIdx.x * 2246822519u);
    x ^= x >> 15;
    x *= 2246822519u;
    x ^= x >> 13;
    if ((x & 7u) == 0) __nanosleep(x % P.jitter_ns);
}

__device__ __forceinline__ void jitter_warp(const Params& P) {
    if (P.jitter_ns == 0) return;
    uint32_t x = (uint32_t)globaltimer() * 2654435761u ^ ((threadIdx.x >> 5) * 40503u) ^ (blockIdx.x * 2246822519u);
    x ^= x >> 15;
    x *= 2246822519u;
    x ^= x >> 13;
    x = __shfl_sync(0xffffffffu, x, 0);
    if ((x & 7u) == 0) __nanosleep(x % P.jitter_ns);
    __syncwarp();
}

// ------------------------------------------------------------------ errors

__device__ __forceinline__ void raise_error(const Params& P, int code) {
    // host-mapped word; plain store (no PCIe atomics needed): every writer stores a nonzero code
    *(volatile int*)P.err = code;
    __threadfence_system();
}

// Spin until *p >= v; false on timeout (error latched).  The spin loop is out
// of line (code size) and takes the few Params fields it needs BY VALUE: passing
// `const Params&` to a non-inlined function takes the kernel parameter's
// address, which makes every thread copy the whole Params block to its local
// stack at kernel entry (measured: +2 us per two-shot call).
static __device__ __noinline__ bool wait_geq_slow(const uint64_t* p, uint64_t v, int sys,
                                                  unsigned long long timeout_ns, int* err) {
    const uint64_t t0 = globaltimer();
    for (uint32_t it = 1;; ++it) {
        if (ld_acquire(p, sys) >= v) return true;
        if ((it & 255) == 0) {
            if (globaltimer() - t0 > timeout_ns) {
                *(volatile int*)err = POLAR_ETIMEOUT;
                __threadfence_system();
                return false;
            }
            if (*(volatile int*)err) return false;   // someone else failed: give up too
        }
    }
}
__device__ __forceinline__ bool wait_geq(const Params& P, const uint64_t* p, uint64_t v) {
    if (ld_acquire(p, P.sys) >= v) return true;
    return wait_geq_slow(p, v, P.sys, P.timeout_ns, P.err);
}

// Poll one LL line until both flags equal `flag`; false on timeout.  The spin is
// out of line with by-value arguments (code size where many polls are inlined,
// and no address of the kernel's Params is taken).
struct PollRes {
    uint4 v;
    int ok;
};
static __device__ __noinline__ PollRes poll_ll_slow(const uint4* p, uint32_t flag, unsigned long long timeout_ns,
                                                   int* err) {
    PollRes r;
    const uint64_t t0 = globaltimer();
    for (uint32_t it = 1;; ++it) {
        r.v = ld_ll(p);
        if (r.v.y == flag && r.v.w == flag) { r.ok = 1; return r; }
        if ((it & 1023) == 0) {
            if (globaltimer() - t0 > timeout_ns) {
                *(volatile int*)err = POLAR_ETIMEOUT;
                __threadfence_system();
                r.ok = 0;
                return r;
            }
            if (*(volatile int*)err) { r.ok = 0; return r; }
        }
    }
}
__device__ __forceinline__ bool poll_ll(const Params& P, const uint4* p, uint32_t flag, uint4& out) {
    uint4 v = ld_ll(p);
    if (v.y == flag && v.w == flag) { out = v; return true; }
    const PollRes r = poll_ll_slow(p, flag, P.timeout_ns, P.err);
    out = r.v;
    return r.ok != 0;
}

// LL128 reader helpers: does this lane's 16 B of a line group carry `flag`
// (only flag lanes check), and the inverse of st_ll128's shuffle (lane L < 30
// gets pack L; lanes 30, 31 get padding).  Both warp-collective (shuffles).
__device__ __forceinline__ bool ll128_lane_ready(const uint4& w, uint64_t flag) {
    return (threadIdx.x & 7) != 7 || (w.z == (uint32_t)flag && w.w == (uint32_t)(flag >> 32));
}
__device__ __forceinline__ uint4 ll128_unpack(const uint4& w) {
    const int lane = (int)(threadIdx.x & 31);
    const int s0 = lane < 28 ? (lane / 7) * 8 + lane % 7 : (lane == 28 ? 7 : 23);
    const int s1 = lane == 29 ? 31 : 15;
    uint4 a;
    a.x = __shfl_sync(0xffffffffu, w.x, s0);
    a.y = __shfl_sync(0xffffffffu, w.y, s0);
    a.z = __shfl_sync(0xffffffffu, w.z, s0);
    a.w = __shfl_sync(0xffffffffu, w.w, s0);
    const uint32_t b0 = __shfl_sync(0xffffffffu, w.x, s1);
    const uint32_t b1 = __shfl_sync(0xffffffffu, w.y, s1);
    return lane < 28 ? a : make_uint4(a.x, a.y, b0, b1);
}

// Poll one LL128 line group until all four flags equal `flag`, then unpack.
// Warp-uniform result; false on timeout (error latched).  Out of line with
// by-value arguments like poll_ll_slow; warp-collective.
static __device__ __noinline__ PollRes ld_ll128_slow(const uint4* group, uint64_t flag, unsigned long long timeout_ns,
                                                    int* err) {
    const int lane = (int)(threadIdx.x & 31);
    PollRes r;
    uint4 w;
    uint64_t t0 = 0;
    for (uint32_t it = 0;; ++it) {
        w = ld_ll(group + lane);
        if (__all_sync(0xffffffffu, ll128_lane_ready(w, flag))) break;
        if ((it & 1023) == 1023) {
            int bad = 0;
            if (lane == 0) {
                const uint64_t now = globaltimer();
                if (t0 == 0) t0 = now;
                if (now - t0 > timeout_ns) {
                    *(volatile int*)err = POLAR_ETIMEOUT;
                    __threadfence_system();
                    bad = 1;
                } else if (*(volatile int*)err) {
                    bad = 1;
                }
            }
            if (__shfl_sync(0xffffffffu, bad, 0)) { r.ok = 0; r.v = w; return r; }
        }
    }
    r.v = ll128_unpack(w);
    r.ok = 1;
    return r;
}
__device__ __forceinline__ bool ld_ll128(const Params& P, const uint4* group, uint64_t flag, uint4& out) {
    const PollRes r = ld_ll128_slow(group, flag, P.timeout_ns, P.err);
    out = r.v;
    return r.ok != 0;
}

// ------------------------------------------------------------ scratch access

__device__ __forceinline__ uint64_t* flag_ptr(const Params& P, int owner, int kind, int ch, int slot) {
    return reinterpret_cast<uint64_t*>(P.scratch[owner] + P.flags_off + ((size_t)kind * kMaxCh + ch) * kFlagRow) +
           slot;
}
__device__ __forceinline__ ChanState* chan_state(const Params& P, int rank, int ch) {
    return reinterpret_cast<ChanState*>(P.scratch[rank] + P.state_off) + ch;
}

// ------------------------------------------------------------------ dtypes

template <int DT> struct DType;
template <> struct DType<POLAR_INT32> { using T = int32_t; static constexpr int ES = 4; };
template <> struct DType<POLAR_INT64> { using T = long long; static constexpr int ES = 8; };
template <> struct DType<POLAR_FLOAT32> { using T = float; static constexpr int ES = 4; };
template <> struct DType<POLAR_BFLOAT16> { using T = __nv_bfloat16; static constexpr int ES = 2; };

// Accumulator of one 16-B pack.  For bf16 it holds 8 f32 partials (32 B on the
// wire: "bf16 reduce-phase partials travel as f32").
template <int DT> struct Acc { uint4 w[1]; };
template <> struct Acc<POLAR_BFLOAT16> { uint4 w[2]; };
template <int DT> struct AccWords { static constexpr int N = 1; };
template <> struct AccWords<POLAR_BFLOAT16> { static constexpr int N = 2; };

__device__ __forceinline__ uint32_t u32_comb(uint32_t a, uint32_t b, int op) {
    if (op == POLAR_SUM) return a + b;   // two's-complement wrap
    int x = (int)a, y = (int)b;
    return (uint32_t)(op == POLAR_MAX ? (x > y ? x : y) : (x < y ? x : y));
}
__device__ __forceinline__ unsigned long long u64_comb(unsigned long long a, unsigned long long b, int op) {
    if (op == POLAR_SUM) return a + b;
    long long x = (long long)a, y = (long long)b;
    return (unsigned long long)(op == POLAR_MAX ? (x > y ? x : y) : (x < y ? x : y));
}
__device__ __forceinline__ float f32_comb(float a, float b, int op) {
    if (op == POLAR_SUM) return __fadd_rn(a, b);   // one RNE add, never contracted
    return op == POLAR_MAX ? fmaxf(a, b) : fminf(a, b);
}
__device__ __forceinline__ uint32_t f32_comb_bits(uint32_t a, uint32_t b, int op) {
    return __float_as_uint(f32_comb(__uint_as_float(a), __uint_as_float(b), op));
}

// acc <- widen(pack)
template <int DT> __device__ __forceinline__ void acc_init(Acc<DT>& a, uint4 p) {
    if constexpr (DT == POLAR_BFLOAT16) {
        a.w[0] = make_uint4(p.x << 16, p.x & 0xFFFF0000u, p.y << 16, p.y & 0xFFFF0000u);
        a.w[1] = make_uint4(p.z << 16, p.z & 0xFFFF0000u, p.w << 16, p.w & 0xFFFF0000u);
    } else {
        a.w[0] = p;
    }
}

// acc <- acc (op) widen(pack)
template <int DT, int OP> __device__ __forceinline__ void acc_add(Acc<DT>& a, uint4 p) {
    if constexpr (DT == POLAR_INT32) {
        a.w[0].x = u32_comb(a.w[0].x, p.x, OP); a.w[0].y = u32_comb(a.w[0].y, p.y, OP);
        a.w[0].z = u32_comb(a.w[0].z, p.z, OP); a.w[0].w = u32_comb(a.w[0].w, p.w, OP);
    } else if constexpr (DT == POLAR_INT64) {
        unsigned long long a0 = ((unsigned long long)a.w[0].y << 32) | a.w[0].x;
        unsigned long long a1 = ((unsigned long long)a.w[0].w << 32) | a.w[0].z;
        unsigned long long b0 = ((unsigned long long)p.y << 32) | p.x;
        unsigned long long b1 = ((unsigned long long)p.w << 32) | p.z;
        a0 = u64_comb(a0, b0, OP); a1 = u64_comb(a1, b1, OP);
        a.w[0] = make_uint4((uint32_t)a0, (uint32_t)(a0 >> 32), (uint32_t)a1, (uint32_t)(a1 >> 32));
    } else if constexpr (DT == POLAR_FLOAT32) {
        a.w[0].x = f32_comb_bits(a.w[0].x, p.x, OP); a.w[0].y = f32_comb_bits(a.w[0].y, p.y, OP);
        a.w[0].z = f32_comb_bits(a.w[0].z, p.z, OP); a.w[0].w = f32_comb_bits(a.w[0].w, p.w, OP);
    } else {
        Acc<DT> b;
        acc_init<DT>(b, p);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            a.w[k].x = f32_comb_bits(a.w[k].x, b.w[k].x, OP); a.w[k].y = f32_comb_bits(a.w[k].y, b.w[k].y, OP);
            a.w[k].z = f32_comb_bits(a.w[k].z, b.w[k].z, OP); a.w[k].w = f32_comb_bits(a.w[k].w, b.w[k].w, OP);
        }
    }
}

// acc <- acc (op) acc2 (both already widened; used when partials meet partials)
template <int DT, int OP> __device__ __forceinline__ void acc_merge(Acc<DT>& a, const Acc<DT>& b) {
    if constexpr (DT == POLAR_BFLOAT16) {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            a.w[k].x = f32_comb_bits(a.w[k].x, b.w[k].x, OP); a.w[k].y = f32_comb_bits(a.w[k].y, b.w[k].y, OP);
            a.w[k].z = f32_comb_bits(a.w[k].z, b.w[k].z, OP); a.w[k].w = f32_comb_bits(a.w[k].w, b.w[k].w, OP);
        }
    } else {
        acc_add<DT, OP>(a, b.w[0]);
    }
}

__device__ __forceinline__ uint32_t bf16x2_rn(uint32_t lo_f32, uint32_t hi_f32) {
    __nv_bfloat16 l = __float2bfloat16_rn(__uint_as_float(lo_f32));
    __nv_bfloat16 h = __float2bfloat16_rn(__uint_as_float(hi_f32));
    return (uint32_t)__bfloat16_as_ushort(l) | ((uint32_t)__bfloat16_as_ushort(h) << 16);
}

// pack <- narrow(acc): the single bf16 rounding (RNE) of every output element
template <int DT> __device__ __forceinline__ uint4 acc_fin(const Acc<DT>& a) {
    if constexpr (DT == POLAR_BFLOAT16) {
        return make_uint4(bf16x2_rn(a.w[0].x, a.w[0].y), bf16x2_rn(a.w[0].z, a.w[0].w),
                          bf16x2_rn(a.w[1].x, a.w[1].y), bf16x2_rn(a.w[1].z, a.w[1].w));
    } else {
        return a.w[0];
    }
}

// ----------------------------------------------------- packs of user data
// The message is a sequence of 16-B packs; the last one may be partial
// (nvalid < 16/ES elements).  Unaligned buffers fall back to element copies.

template <int ES> __device__ __forceinline__ int pack_valid(unsigned long long count, unsigned long long idx) {
    constexpr unsigned long long V = 16 / ES;
    unsigned long long rem = count - idx * V;
    return rem >= V ? (int)V : (int)rem;
}

template <int ES> __device__ __forceinline__ uint4 load_pack_slow(const char* base, unsigned long long idx, int nvalid) {
    uint4 r = make_uint4(0, 0, 0, 0);
    char* rb = reinterpret_cast<char*>(&r);
    const char* src = base + idx * 16;
    for (int i = 0; i < nvalid; ++i) {
        if constexpr (ES == 2) reinterpret_cast<uint16_t*>(rb)[i] = reinterpret_cast<const uint16_t*>(src)[i];
        else if constexpr (ES == 4) reinterpret_cast<uint32_t*>(rb)[i] = reinterpret_cast<const uint32_t*>(src)[i];
        else reinterpret_cast<unsigned long long*>(rb)[i] = reinterpret_cast<const unsigned long long*>(src)[i];
    }
    return r;
}
template <int ES> __device__ __forceinline__ void store_pack_slow(char* base, unsigned long long idx, uint4 v, int nvalid) {
    const char* vb = reinterpret_cast<const char*>(&v);
    char* dst = base + idx * 16;
    for (int i = 0; i < nvalid; ++i) {
        if constexpr (ES == 2) reinterpret_cast<uint16_t*>(dst)[i] = reinterpret_cast<const uint16_t*>(vb)[i];
        else if constexpr (ES == 4) reinterpret_cast<uint32_t*>(dst)[i] = reinterpret_cast<const uint32_t*>(vb)[i];
        else reinterpret_cast<unsigned long long*>(dst)[i] = reinterpret_cast<const unsigned long long*>(vb)[i];
    }
}

// load pack idx of a user buffer (own or peer); .cg keeps peer data out of L1
template <int ES> __device__ __forceinline__ uint4 load_pack(const Params& P, const char* base, unsigned long long idx) {
    int nv = pack_valid<ES>(P.count, idx);
    if (P.vec && nv == 16 / ES) return ld_cg(reinterpret_cast<const uint4*>(base) + idx);
    return load_pack_slow<ES>(base, idx, nv);
}
template <int ES> __device__ __forceinline__ void store_pack(const Params& P, char* base, unsigned long long idx, uint4 v) {
    int nv = pack_valid<ES>(P.count, idx);
    if (P.vec && nv == 16 / ES) { st_plain(reinterpret_cast<uint4*>(base) + idx, v); return; }
    store_pack_slow<ES>(base, idx, v, nv);
}

// ------------------------------------------------------------ partitioning
// Ranges of packs in 32-pack (512 B) units so that shards/slices start on 512 B.
constexpr unsigned long long kUnit = 32;

__device__ __forceinline__ void split_range(unsigned long long lo, unsigned long long hi, int parts, int k,
                                            unsigned long long& a, unsigned long long& b) {
    unsigned long long units = (hi - lo + kUnit - 1) / kUnit;
    unsigned long long ua = units * (unsigned long long)k / (unsigned long long)parts;
    unsigned long long ub = units * (unsigned long long)(k + 1) / (unsigned long long)parts;
    a = lo + ua * kUnit;
    b = lo + ub * kUnit;
    if (a > hi) a = hi;
    if (b > hi) b = hi;
}

}  // namespace dev
}  // namespace polar
