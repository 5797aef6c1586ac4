// Ring and tree Simple for VIRTUAL comms as thread-block clusters (SURVEY.md §8
// rows a4, a6, a8, a9; DESIGN.md §8 "Cluster transport").
//
// A virtual comm hosts all n ranks on one GPU.  The FIFO kernels (kernels.cuh
// ring / ring_simple_ws / tree_simple_ws) move every hop through a FIFO in HBM
// (L2), so on one GPU the ring issues 6n - 4 memory operations of S/n per rank
// against the two-shot's 2: it is bound by that memory-operation count, not by
// its wires.  Here the n ranks of one channel are the n CTAs of ONE cluster
// (cluster rank = rank), and a hop is a distributed-shared-memory store into the
// receiver's shared-memory inbox:
//   * the sender's warps write the tile with st.async (16 B per lane) straight
//     into the receiver's inbox stage; each warp also arrives on the receiver's
//     `full` mbarrier with the byte count it sent (expect_tx), so the phase
//     completes exactly when every byte of the tile has landed;
//   * the receiver's warps read the stage, then arrive on the sender's `empty`
//     mbarrier (remote arrive, release.cluster): the stage may be rewritten;
//   * a loader warp streams the rank's own input tiles from HBM into shared
//     memory with cp.async.bulk (TMA), as far ahead as its stages allow — own
//     data does not depend on the ring;
//   * results go to HBM with 16-B stores from registers.
// HBM then sees each input read once and each output written once: 2 n S per
// call, the same algorithmic bytes as the two-shot.  The schedule, the chunk
// geometry and the reduction order are the FIFO ring's / tree's, so for the
// same channel count the results are bit-identical to the FIFO kernels
// (GPU test test_cluster_matches_fifo).
//
// The cluster's CTAs are co-scheduled by the hardware, so no wait here depends
// on another launch or on co-residency; every wait is still bounded
// (POLAR_ETIMEOUT latched, then an orderly exit).  Channels are independent
// clusters.  Real comms (ranks on different GPUs) keep the FIFO kernels: a
// cluster cannot span GPUs.
//
// Used when every pack is a whole 16-B pack of a 16-B aligned buffer (bulk copies
// are 16-B granular); otherwise the FIFO kernels run.
#pragma once
#include "kernels.cuh"   // npacks, split_range, Acc arithmetic (device.cuh)

namespace polar {
namespace dev {

// POLAR_CL_AGL2=1: the ring's all-gather through L2 instead of DSMEM (pull
// from the predecessor's buffer with TMA; DESIGN.md §8 "Cluster transport",
// measured variant).  Correct (the cluster GPU tests pass with it) but slower
// on 8 x 128 MiB: f32 739 vs 685 us, bf16 1413 vs 926 us — two pull stages of
// shared memory hold too few bytes in flight for the L2 round trip, and the
// reduce-scatter inbox needs the rest of the 227 KB.  Off by default.
#ifndef POLAR_CL_AGL2
#define POLAR_CL_AGL2 0
#endif
#ifndef POLAR_CL_WARPS
#define POLAR_CL_WARPS 8          // compute warps (warp 0 loads, warp 1 signals, [last: all-gather])
#endif
#ifndef POLAR_CL_STAGES
#if POLAR_CL_AGL2
#define POLAR_CL_STAGES 8         // ring inbox stages (>= tiles per ring step + slack)
#else
#define POLAR_CL_STAGES 10
#endif
#endif
#ifndef POLAR_CL_SLACK
#define POLAR_CL_SLACK (POLAR_CL_AGL2 ? 2 : 3)   // inbox stages beyond one ring step (4: 650 us, 3: 645 us f32; 896 / 885 bf16)
#endif
#ifndef POLAR_CL_AGP
#define POLAR_CL_AGP 2            // all-gather pull stages (POLAR_CL_AGL2)
#endif
#ifndef POLAR_CL_AGF
#define POLAR_CL_AGF 2            // final-tile stages (POLAR_CL_AGL2)
#endif
#ifndef POLAR_CL_AGLAG
#define POLAR_CL_AGLAG 1          // pull stores in flight before a tile is published
#endif
#ifndef POLAR_CL_MINB
#define POLAR_CL_MINB 1           // CTAs per SM the register budget is sized for
#endif
#ifndef POLAR_CL_OWN
#if POLAR_CL_AGL2
#define POLAR_CL_OWN 2            // own-input stages (TMA loads in flight)
#else
#define POLAR_CL_OWN 4            // (3: 128 MiB f32 685 us, 4: 650 us; profiles/r02y_cluster_ring_ab.jsonl)
#endif
#endif
#ifndef POLAR_CL_JITTER
#define POLAR_CL_JITTER 1         // fault injection point in the ring's tile loop (0 off, 1 before, 2 after the sends)
#endif
#ifndef POLAR_CL_PF
#define POLAR_CL_PF 0             // own tiles prefetched into L2 ahead of the TMA loads (0: off)
#endif
constexpr int kClPf = POLAR_CL_PF;
constexpr int kClWarps = POLAR_CL_WARPS;
constexpr bool kClAgL2 = POLAR_CL_AGL2 != 0;
constexpr int kClAgP = kClAgL2 ? POLAR_CL_AGP : 0;
constexpr int kClAgF = kClAgL2 ? POLAR_CL_AGF : 0;
constexpr int kClAg = kClAgP + kClAgF;
constexpr int kClAgLag = POLAR_CL_AGLAG;
constexpr int kClThreads = 32 * (kClWarps + 2 + (kClAgL2 ? 2 : 0));
constexpr int kClStages = POLAR_CL_STAGES;
constexpr int kClOwn = POLAR_CL_OWN;
#ifndef POLAR_CL_WIRE
#define POLAR_CL_WIRE 1024        // 16-B wire words per stage (16 KiB)
#endif
constexpr unsigned kClWire = POLAR_CL_WIRE;
constexpr size_t kClStageBytes = (size_t)kClWire * 16;
// element packs per tile: a tile's wire words fill one stage (bf16: 2 f32 words per pack)
template <int AW> __host__ __device__ constexpr unsigned cl_tile() { return kClWire / (unsigned)AW; }
// ring inbox stages needed per ring step + slack for the credit round trip
constexpr int kClSlack = POLAR_CL_SLACK;
__host__ __device__ constexpr size_t cl_ring_smem_bytes() {
    return (size_t)(kClStages + kClOwn + kClAg) * kClStageBytes +
           (size_t)(3 * kClStages + 2 * kClOwn + kClAg + 3) * 8;
}

// ----------------------------------------------------------- cluster primitives
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// this CTA's shared address `a` as seen in cluster CTA `rank`'s shared window
__device__ __forceinline__ uint32_t cl_map(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void cl_st_async(uint32_t raddr, uint4 v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%2,%3,%4}, [%5];" ::"r"(raddr),
                 "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rbar)
                 : "memory");
}
// Remote arrives are RELAXED: a release arrive makes the issuing thread wait
// until its earlier global stores (the results just written to HBM) are
// performed at cluster scope, ~1 us per tile on the critical path.  No release
// is needed: `full` carries its data through st.async's complete_tx, and an
// `empty` credit follows shared-memory reads whose values were already
// consumed (stored / sent) by the warp before its __syncwarp.
#ifndef POLAR_CL_RELEASE
#define POLAR_CL_RELEASE 0
#endif
#if POLAR_CL_RELEASE
#define POLAR_CL_SEM "release"
#else
#define POLAR_CL_SEM "relaxed"
#endif
__device__ __forceinline__ void cl_arrive_remote(uint32_t rbar) {
    asm volatile("mbarrier.arrive." POLAR_CL_SEM ".cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
}
__device__ __forceinline__ void cl_arrive_expect_remote(uint32_t rbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx." POLAR_CL_SEM ".cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(rbar),
                 "r"(bytes)
                 : "memory");
}
// Waits are acquire.CTA (the default): acquire.cluster compiles to a
// CCTL.IVALL (whole-L1 invalidation) after every successful wait, which the
// compute warps paid once per tile.  Nothing here reads global memory that a
// peer wrote through the generic proxy: inbox data arrives through st.async,
// whose bytes are complete when the mbarrier phase completes (complete_tx),
// and credits order nothing but shared-memory reuse.  (Measured:
// mbarrier.test_wait spinning and try_wait with an explicit suspend-time hint
// were no faster; profiles/r02t_cluster_wait_variants.jsonl.)
__device__ __forceinline__ bool cl_try_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, "
        "p;\n}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ uint4 ld_shared_v4(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
// Bounded wait for the completion of the phase with parity `parity`.  `honour_err`:
// give up as soon as another thread latched an error (the final rendezvous
// waits for its peers regardless, so that no CTA leaves while a peer may still
// write its shared memory).
static __device__ __noinline__ bool cl_wait_slow(uint32_t bar, uint32_t parity, unsigned long long timeout_ns, int* err,
                                                 int honour_err) {
    const uint64_t t0 = globaltimer();
    for (uint32_t it = 1;; ++it) {
        if (cl_try_wait(bar, parity)) return true;
        if ((it & 63) == 0) {
            if (globaltimer() - t0 > timeout_ns) {
                *(volatile int*)err = POLAR_ETIMEOUT;
                __threadfence_system();
                return false;
            }
            if (honour_err && *(volatile int*)err) return false;
        }
    }
}
__device__ __forceinline__ bool cl_wait(const Params& P, uint32_t bar, uint32_t parity) {
    if (cl_try_wait(bar, parity)) return true;
    return cl_wait_slow(bar, parity, P.timeout_ns, P.err, 1);
}
// Bounded wait until the u32 at shared address `a` (a monotone count) is >= v.
static __device__ __noinline__ bool cl_wait_count_slow(uint32_t a, uint32_t v, unsigned long long timeout_ns, int* err) {
    const uint64_t t0 = globaltimer();
    for (uint32_t it = 1;; ++it) {
        uint32_t c;
        asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(c) : "r"(a) : "memory");
        if (c >= v) return true;
        if ((it & 63) == 0) {
            if (globaltimer() - t0 > timeout_ns) {
                *(volatile int*)err = POLAR_ETIMEOUT;
                __threadfence_system();
                return false;
            }
            if (*(volatile int*)err) return false;
        }
    }
}
__device__ __forceinline__ bool cl_wait_count(const Params& P, uint32_t a, uint32_t v) {
    uint32_t c;
    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(c) : "r"(a) : "memory");
    if (c >= v) return true;
    return cl_wait_count_slow(a, v, P.timeout_ns, P.err);
}

// Shared memory of one cluster-ring CTA (dynamic; byte offsets):
//   inbox [kClStages][kClStageBytes]  written by the predecessor (st.async)
//   own   [kClOwn][kClStageBytes]     my input tiles (TMA)
//   full  [kClStages]  inbox stage landed: 1 arrival (my signal warp arms it with
//                      the tile's byte count) + the predecessor's st.async bytes
//   cons  [kClStages]  my compute warps have read the stage (kClWarps arrivals)
//   empty [kClStages]  the successor's stage is free: 1 remote arrival (its
//                      signal warp, after its cons)
//   ofull [kClOwn]     own tile landed (1 arrival + tx; loader)
//   oempty[kClOwn]     own stage free (kClWarps arrivals)
//   fin                final rendezvous (n - 1 remote arrivals)
// Inbox words are planar: word q of element pack p of a tile at (q * TP + p) * 16,
// so a warp's 16-B accesses are contiguous (no 32-B stride bank conflicts).
// Compute warps only touch local barriers; the one remote arrive per tile (the
// credit) is the signal warp's, off the data path.
// With POLAR_CL_AGL2 (all-gather through L2):
//   agst  [kClAgF + kClAgP][kClStageBytes]  final tiles, then pulled tiles, on
//                  their way to my buffer
//   finfull[kClAgF] my compute warps wrote a final tile into the stage (kClWarps arrivals)
//   loaded [kClAgP] the predecessor's tile landed (1 arrival + tx; pull warp)
//   cnt            tiles the predecessor has published in its buffer (u32,
//                  written by the predecessor's pull warp)
//   finok          final tiles whose stage the store warp has handed out (u32)
//   findone        final tiles whose stores completed (u32, store warp -> pull warp)
struct ClRingSmem {
    uint32_t inbox, own, full, cons, empty, ofull, oempty, fin;
    uint32_t agst, finfull, loaded, cnt, finok, findone;
};
__device__ __forceinline__ ClRingSmem cl_ring_smem(uint32_t base) {
    ClRingSmem s;
    s.inbox = base;
    s.own = base + (uint32_t)(kClStages * kClStageBytes);
    s.agst = s.own + (uint32_t)(kClOwn * kClStageBytes);
    s.full = s.agst + (uint32_t)(kClAg * kClStageBytes);
    s.cons = s.full + 8u * kClStages;
    s.empty = s.cons + 8u * kClStages;
    s.ofull = s.empty + 8u * kClStages;
    s.oempty = s.ofull + 8u * kClOwn;
    s.finfull = s.oempty + 8u * kClOwn;
    s.loaded = s.finfull + 8u * kClAgF;
    s.fin = s.loaded + 8u * kClAgP;
    s.cnt = s.fin + 8u;
    s.finok = s.cnt + 4u;
    s.findone = s.finok + 4u;
    return s;
}
__device__ __forceinline__ void mbar_init_u32(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_u32(uint32_t bar) {
    asm volatile("mbarrier.arrive." POLAR_CL_SEM ".cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// release (CTA scope): my shared-memory writes before it are visible to the waiter
__device__ __forceinline__ void mbar_arrive_rel_u32(uint32_t bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_u32(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx." POLAR_CL_SEM ".cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_load_u32(uint32_t sdst, const void* gsrc, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sdst),
                 "l"(gsrc), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Final rendezvous: no CTA leaves while a peer may still touch its shared memory
// (the successor's last credits land on my `empty` barriers after my loop).
// Thread 0 of each CTA arrives on every peer's `fin` and waits for its own.
// The fence matters: every warp's remote operations (credits on a peer's
// barriers, published counts, st.async) precede the __syncthreads, and the
// cluster-scope fence orders them before the fin arrives — a relaxed fin
// arrive could otherwise overtake, say, the signal warp's last credit, the
// peer could leave, and the late credit would land in the shared memory of
// the next kernel's CTA on that SM (compute-sanitizer memcheck caught the
// resulting launch failure in a back-to-back sequence).
__device__ __forceinline__ void cl_rendezvous(const Params& P, uint32_t fin, int r, int n) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        for (int p = 0; p < n; ++p)
            if (p != r) cl_arrive_remote(cl_map(fin, (uint32_t)p));
        // (3x the loop timeout: a straggler that timed out in its loop arrives
        // up to one timeout late; giving up at the same moment would let this
        // CTA leave just before the straggler's fin arrive lands in it)
        if (!cl_try_wait(fin, 0)) cl_wait_slow(fin, 0, 3 * P.timeout_ns, P.err, 0);
    }
    __syncthreads();
}

// The ring schedule of one channel, exactly as kernels.cuh `ring` walks it:
// laps of n sub-chunks of SP packs; step s of 2(n-1)+1 handles sub-chunk k(s);
// each sub-chunk in tiles of TP packs.  A resumable cursor, so that the signal
// warp can walk the received tiles kClStages ahead of its own position.
struct RingCursor {
    unsigned long long base, L, ks, ke, i0;
    int s;
    bool done;
};
__device__ __forceinline__ void ring_cursor_step(RingCursor& q, int r, int n, unsigned long long cb,
                                                 unsigned long long SP) {
    // position q at the first tile of step q.s of the lap at q.base (or later)
    const unsigned long long LC = SP * (unsigned long long)n;
    for (;;) {
        if (q.base >= cb) { q.done = true; return; }
        q.L = (cb - q.base < LC) ? cb - q.base : LC;
        if (q.s > 2 * (n - 1)) { q.base += LC; q.s = 0; continue; }
        int k;
        if (q.s < n) k = ((r - q.s) % n + n) % n;
        else k = ((r - (q.s - n)) % n + n) % n;
        if (q.s == n - 1) k = (r + 1) % n;
        q.ks = q.base + q.L * (unsigned long long)k / n;
        q.ke = q.base + q.L * (unsigned long long)(k + 1) / n;
        q.i0 = q.ks;
        if (q.ks < q.ke) return;
        ++q.s;   // empty sub-chunk (tiny lap): no tile
    }
}
__device__ __forceinline__ RingCursor ring_cursor(int r, int n, unsigned long long ca, unsigned long long cb,
                                                  unsigned long long SP) {
    RingCursor q;
    q.base = ca;
    q.s = 0;
    q.done = false;
    ring_cursor_step(q, r, n, cb, SP);
    return q;
}
__device__ __forceinline__ unsigned ring_cursor_npk(const RingCursor& q, unsigned TP) {
    return (unsigned)((q.ke - q.i0) < TP ? (q.ke - q.i0) : TP);
}
__device__ __forceinline__ void ring_cursor_next(RingCursor& q, int r, int n, unsigned long long cb,
                                                 unsigned long long SP, unsigned TP) {
    q.i0 += TP;
    if (q.i0 < q.ke) return;
    ++q.s;
    ring_cursor_step(q, r, n, cb, SP);
}
template <class F>
__device__ __forceinline__ bool cl_ring_walk(int r, int n, unsigned long long ca, unsigned long long cb,
                                             unsigned long long SP, unsigned TP, F&& f) {
    for (RingCursor q = ring_cursor(r, n, ca, cb, SP); !q.done; ring_cursor_next(q, r, n, cb, SP, TP))
        if (!f(q.s, q.i0, ring_cursor_npk(q, TP))) return false;
    return true;
}
// next RECEIVED tile (steps s >= 1) at or after q
__device__ __forceinline__ void ring_cursor_recv(RingCursor& q, int r, int n, unsigned long long cb,
                                                 unsigned long long SP, unsigned TP) {
    // (all-gather through L2: only the reduce-scatter steps 1..n-1 receive via DSMEM)
    while (!q.done && (q.s == 0 || (kClAgL2 && q.s >= n))) ring_cursor_next(q, r, n, cb, SP, TP);
}
// next all-gather item (POLAR_CL_AGL2): the final step's tiles (s = n-1,
// produced by my compute warps) and the all-gather steps' tiles (s >= n,
// pulled from the predecessor's buffer), in walk order
__device__ __forceinline__ void ring_cursor_ag(RingCursor& q, int r, int n, unsigned long long cb,
                                               unsigned long long SP, unsigned TP) {
    while (!q.done && q.s < n - 1) ring_cursor_next(q, r, n, cb, SP, TP);
}

// Sub-chunk size: the FIFO ring's slot (same geometry => same reduction order),
// capped so that one ring step fits the inbox with kClSlack stages to spare.
// (Each rank receives a whole step before its successor frees it: a ring step
// must fit the inbox or the ring deadlocks.)
template <int AW> __device__ __forceinline__ unsigned long long cl_ring_sp(const Params& P) {
    const unsigned long long fifo = P.ring_slot / 16 / AW;
    const unsigned long long cap = (unsigned long long)(kClStages - kClSlack) * cl_tile<AW>();
    return fifo < cap ? fifo : cap;
}

// Step kinds of the ring schedule (uniform per step):
//   first  s = 0        own -> [widen] -> successor              (AW words)
//   mid    0 < s < n-1  inbox (AW) (op) own -> successor         (AW words)
//   fin    s = n-1      fin(inbox (op) own) -> HBM + successor  (1 word)
//   ag     n-1 < s < 2(n-1)   inbox (1) -> HBM + successor
//   last   s = 2(n-1)   inbox (1) -> HBM
enum { kClFirst = 0, kClMid = 1, kClFin = 2, kClAgStep = 3, kClLast = 4 };

// The compute warps' state and per-step tile loop.  Stage indices and phase
// parities are 32-bit counters that wrap (no 64-bit division per tile); each
// step kind is its own instantiation, so the per-pack code has no step branches.
template <int DT, int OP>
struct ClCompute {
    static constexpr int AW = AccWords<DT>::N;
    static constexpr unsigned TP = cl_tile<AW>();
    static constexpr unsigned NT = kClWarps * 32;             // compute threads
    static constexpr unsigned PPL = (TP + NT - 1) / NT;       // packs per lane per tile
    ClRingSmem S;
    uint32_t dst_inbox, dst_full;
    uint4* mine;
    uint32_t me;                                              // compute thread index
    uint32_t xi = 0, pi = 0;        // inbox stage / parity of the phase to wait for
    uint32_t xo = 0, pe = 1;        // successor stage / parity of its credit phase
    uint32_t xw = 0, pw = 0;        // own stage / parity
    bool wrapped = false;           // sent >= kClStages: credits are needed
    unsigned long long ag_item = 0; // POLAR_CL_AGL2: final tiles staged so far

    // One tile: every shared-memory load of the lane's PPL packs first, then
    // the arithmetic, then the stores (one register set per pack: loads of later
    // packs are not serialised behind the stores of earlier ones).
    // (POLAR_CL_AGL2, final step: `dst` is the local all-gather stage; the
    // result goes there, and the all-gather warp stores it and publishes it)
    template <int KIND, bool FULL>
    __device__ __forceinline__ void body(uint32_t in, uint32_t ow, uint32_t dst, uint32_t dbar, uint4* gout,
                                         unsigned npk) {
        constexpr bool STAGE = kClAgL2 && KIND == kClFin;
        constexpr bool SEND = KIND != kClLast && !STAGE, OWN = KIND <= kClFin, OUT = KIND >= kClFin && !STAGE;
        constexpr int WIN = (KIND == kClMid || KIND == kClFin) ? AW : (KIND == kClFirst ? 0 : 1);
        constexpr int WOUT = KIND <= kClMid ? AW : 1;
        uint4 o[PPL], a[PPL][AW > 1 ? AW : 1];
#pragma unroll
        for (unsigned u = 0; u < PPL; ++u) {
            const unsigned p = u * NT + me;
            if ((!FULL || TP % NT != 0) && p >= npk) continue;   // (a warp count that does not divide TP)
            if constexpr (OWN) o[u] = ld_shared_v4(ow + p * 16u);
#pragma unroll
            for (int q = 0; q < WIN; ++q) a[u][q] = ld_shared_v4(in + ((unsigned)q * TP + p) * 16u);
        }
#pragma unroll
        for (unsigned u = 0; u < PPL; ++u) {
            const unsigned p = u * NT + me;
            if ((!FULL || TP % NT != 0) && p >= npk) continue;   // (a warp count that does not divide TP)
            uint4 v = make_uint4(0, 0, 0, 0);
            if constexpr (OWN) {
                Acc<DT> acc;
                if constexpr (KIND == kClFirst) {
                    acc_init<DT>(acc, o[u]);
                } else {
#pragma unroll
                    for (int q = 0; q < AW; ++q) acc.w[q] = a[u][q];
                    acc_add<DT, OP>(acc, o[u]);
                }
                if constexpr (KIND != kClFin) {
#pragma unroll
                    for (int q = 0; q < WOUT; ++q) cl_st_async(dst + ((unsigned)q * TP + p) * 16u, acc.w[q], dbar);
                    continue;
                } else {
                    v = acc_fin<DT>(acc);
                }
            } else {
                v = a[u][0];
            }
            if constexpr (STAGE)
                asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(dst + p * 16u), "r"(v.x), "r"(v.y),
                             "r"(v.z), "r"(v.w)
                             : "memory");
            if constexpr (OUT) {
                st_plain(gout + p, v);
            }
            if constexpr (SEND) cl_st_async(dst + p * 16u, v, dbar);
        }
    }

    template <int KIND>
    __device__ __forceinline__ bool tiles(const Params& P, unsigned long long ks, unsigned long long ke) {
        constexpr bool STAGE = kClAgL2 && KIND == kClFin;
        constexpr bool RECV = KIND != kClFirst, SEND = KIND != kClLast && !STAGE;
        constexpr bool OWN = KIND <= kClFin;
        for (unsigned long long i0 = ks; i0 < ke; i0 += TP) {
            const unsigned npk = (unsigned)((ke - i0) < TP ? (ke - i0) : TP);
            if (RECV && !cl_wait(P, S.full + 8u * xi, pi)) return false;
            if (OWN && !cl_wait(P, S.ofull + 8u * xw, pw)) return false;
            // The credit.  Every sender warp also arrives on the successor's
            // `full` barrier after its tile (below), so the successor cannot
            // consume tile t — and credit stage t mod D again — before every one
            // of my warps has passed its credit wait for tile t.  Without those
            // arrivals a warp with no packs in a short tile could fall a whole
            // stage reuse behind the credits, and its parity wait on `empty`
            // would alias the phase it wants with the one after it and wait for
            // a credit that never comes (found by tests/test_gpu_stress.py:
            // n = 8, a few packs per sub-chunk, fault-injection delays).
            if (SEND && wrapped && !cl_wait(P, S.empty + 8u * xo, pe)) return false;
            uint32_t xa = 0;
            if constexpr (STAGE) {
                // the store warp has handed this final tile its stage (the
                // stage's previous tile has been read by its bulk store)
                xa = (uint32_t)(ag_item % (kClAgF > 0 ? kClAgF : 1));
                if (!cl_wait_count(P, S.finok, (uint32_t)(ag_item + 1))) return false;
            }
            const uint32_t in = S.inbox + xi * (uint32_t)kClStageBytes;
            const uint32_t ow = S.own + xw * (uint32_t)kClStageBytes;
            const uint32_t dst = STAGE ? S.agst + xa * (uint32_t)kClStageBytes : dst_inbox + xo * (uint32_t)kClStageBytes;
            const uint32_t dbar = dst_full + 8u * xo;
            uint4* gout = mine + i0;
            if (SEND && POLAR_CL_JITTER == 1) jitter_warp(P);
            if (npk == TP) body<KIND, true>(in, ow, dst, dbar, gout, npk);
            else body<KIND, false>(in, ow, dst, dbar, gout, npk);
            if (SEND && POLAR_CL_JITTER == 2) jitter_warp(P);
            if constexpr (STAGE) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // -> the bulk store
            __syncwarp();
            if ((me & 31u) == 0) {
                if (RECV) mbar_arrive_u32(S.cons + 8u * xi);   // my reads of the inbox stage are done
                if (SEND) cl_arrive_remote(dbar);   // this warp is past the tile's credit wait
                if (OWN) mbar_arrive_u32(S.oempty + 8u * xw);
                if (STAGE) mbar_arrive_rel_u32(S.finfull + 8u * xa);
            }
            if (STAGE) ++ag_item;
            if (RECV && ++xi == (uint32_t)kClStages) { xi = 0; pi ^= 1u; }
            if (OWN && ++xw == (uint32_t)kClOwn) { xw = 0; pw ^= 1u; }
            if (SEND && ++xo == (uint32_t)kClStages) { xo = 0; pe ^= 1u; wrapped = true; }
        }
        return true;
    }
};

// All-gather through L2 (POLAR_CL_AGL2; DESIGN.md §8 "Cluster transport").
// The ring's all-gather forwards each final sub-chunk from rank to rank; here a
// hop is a pull: at all-gather step s I copy sub-chunk k(s) from my
// predecessor's buffer — where it stored that sub-chunk one step earlier — to
// mine, with a TMA load into a shared-memory stage and a TMA store out of it.
// The final step's tiles come from my compute warps through the same stages.
// After a tile's store has completed (bulk async-group) I publish it: a
// release store of "tiles readable in my buffer" into my successor's shared
// memory, which its all-gather warp polls before pulling.  DSMEM then carries
// only the reduce-scatter partials; the all-gather moves through L2, where my
// predecessor's tiles were just written.  Lane 0 drives the pipeline; the warp
// stays converged.
__device__ __forceinline__ uint32_t cl_ld_acquire_u32(uint32_t a) {
    uint32_t v;
#if POLAR_CL_PUBREL
    asm volatile("ld.acquire.cluster.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
#else
    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
#endif
    return v;
}
// Publication of all-gather tiles: a relaxed store of the count into the
// successor's shared memory, after the tiles' bulk stores have completed
// (cp.async.bulk.wait_group: the writes are performed in L2, where the
// successor's bulk loads read them).  A release store / acquire load at
// cluster scope was measured at ~75 us per publication (it drains far more
// than this thread's completed stores; 8 MiB 27.7 -> 3.8 ms) — the ordering it
// would add is already given by the completed bulk group.
#ifndef POLAR_CL_PUBREL
#define POLAR_CL_PUBREL 0
#endif
#ifndef POLAR_CL_PUBFENCE
#define POLAR_CL_PUBFENCE 0
#endif
__device__ __forceinline__ void cl_st_release_remote_u32(uint32_t ra, uint32_t v) {
#if POLAR_CL_PUBREL
    asm volatile("st.release.cluster.shared::cluster.u32 [%0], %1;" ::"r"(ra), "r"(v) : "memory");
#else
    asm volatile("st.relaxed.cluster.shared::cluster.u32 [%0], %1;" ::"r"(ra), "r"(v) : "memory");
#endif
}
__device__ __forceinline__ void bulk_store_u32(void* gdst, uint32_t ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(ssrc), "r"(bytes)
                 : "memory");
}
// final tiles (step n-1) in walk order: stage in my compute warps' hands ->
// bulk store into my buffer; hands the stage back once its store has read it;
// publishes "final tiles stored" (findone) for the pull warp's prefix count
template <int AW>
__device__ __noinline__ void cl_ring_fin_warp(const Params& P, const ClRingSmem S, int r, int n, unsigned long long ca,
                                              unsigned long long cb, unsigned long long SP, uint4* mine, int lane) {
    constexpr unsigned TP = cl_tile<AW>();
    constexpr int F = kClAgF > 0 ? kClAgF : 1;
    RingCursor q = ring_cursor(r, n, ca, cb, SP);
    uint32_t j = 0;
    for (;;) {
        while (!q.done && q.s != n - 1) ring_cursor_next(q, r, n, cb, SP, TP);
        if (q.done) break;
        const uint32_t x = j % F;
        if (!__all_sync(0xffffffffu, cl_wait(P, S.finfull + 8u * x, (j / F) & 1u))) break;
        if (lane == 0) {
            bulk_store_u32(mine + q.i0, S.agst + x * (uint32_t)kClStageBytes, ring_cursor_npk(q, TP) * 16u);
            bulk_commit();
            bulk_wait_read<0>();   // the stage may be refilled
            asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(S.finok), "r"(j + 1 + F) : "memory");
            // completed stores: all of them if the next tile is not ready yet, else all but this one
            const bool idle = !cl_try_wait(S.finfull + 8u * ((j + 1) % F), ((j + 1) / F) & 1u);
            if (idle) bulk_wait_all();
            else bulk_wait_group<1>();
            asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(S.findone), "r"(idle ? j + 1 : j) : "memory");
        }
        __syncwarp();
        ++j;
        ring_cursor_next(q, r, n, cb, SP, TP);
    }
    if (lane == 0) {
        bulk_wait_all();
        asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(S.findone), "r"(j) : "memory");
    }
    __syncwarp();
}

// Walk-order publication: how many of my readable tiles (final tiles and the
// pulled tiles of steps n .. 2n-3, lap by lap in walk order) are in my buffer,
// given the final tiles stored (fdone) and the pulled tiles stored (pdone).
struct PubCursor {
    RingCursor q;
    uint32_t fi = 0, pi = 0, readable = 0;
    __device__ __forceinline__ void advance(int r, int n, unsigned long long cb, unsigned long long SP, unsigned TP,
                                            uint32_t fdone, uint32_t pdone) {
        for (;;) {
            while (!q.done && q.s < n - 1) ring_cursor_next(q, r, n, cb, SP, TP);
            if (q.done) return;
            if (q.s == n - 1) {
                if (fi >= fdone) return;
                ++fi;
                ++readable;
            } else {
                if (pi >= pdone) return;
                ++pi;
                if (q.s <= 2 * (n - 1) - 1) ++readable;
            }
            ring_cursor_next(q, r, n, cb, SP, TP);
        }
    }
};

// pulled tiles (steps n .. 2(n-1)) in walk order: wait until the predecessor
// published the tile, bulk load it from the predecessor's buffer into a stage,
// bulk store it into mine; publish the walk-order prefix to the successor
template <int AW>
__device__ __noinline__ void cl_ring_pull_warp(const Params& P, const ClRingSmem S, int r, int n,
                                               unsigned long long ca, unsigned long long cb, unsigned long long SP,
                                               uint4* mine, const uint4* pred_buf, uint32_t succ_cnt, int lane) {
    constexpr unsigned TP = cl_tile<AW>();
    constexpr int A = kClAgP > 0 ? kClAgP : 1;
    constexpr int LAG = kClAgLag;
    auto next_pull = [&](RingCursor& c) {
        while (!c.done && c.s < n) ring_cursor_next(c, r, n, cb, SP, TP);
    };
    RingCursor ci = ring_cursor(r, n, ca, cb, SP), cs = ci;   // issue / store cursors
    next_pull(ci);
    next_pull(cs);
    PubCursor pub;
    pub.q = ring_cursor(r, n, ca, cb, SP);
    uint32_t m_iss = 0, m_sto = 0, seen = 0, published = 0, ldpar = 0;
    unsigned long long t0 = 0;
    uint32_t spins = 0;
    bool ok = true;
    auto publish = [&](uint32_t pdone) {
        uint32_t fdone = 0;
        if (lane == 0) asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(fdone) : "r"(S.findone) : "memory");
        fdone = __shfl_sync(0xffffffffu, fdone, 0);
        pub.advance(r, n, cb, SP, TP, fdone, pdone);
        if (pub.readable != published) {
            if (lane == 0) cl_st_release_remote_u32(succ_cnt, pub.readable);
            published = pub.readable;
        }
        __syncwarp();
    };
    while (ok) {
        // ---- issue loads ahead, as the predecessor's count allows
        while (!ci.done && m_iss < m_sto + A) {
            if (seen < m_iss + 1) {
                uint32_t v = 0;
                if (lane == 0) v = cl_ld_acquire_u32(S.cnt);
                seen = __shfl_sync(0xffffffffu, v, 0);
                if (seen < m_iss + 1) break;
            }
            const uint32_t y = m_iss % A;
            if (lane == 0) {
                if (m_iss >= (uint32_t)A) bulk_wait_read<0>();   // the stage's previous store has read it
                const unsigned npk = ring_cursor_npk(ci, TP);
                mbar_expect_u32(S.loaded + 8u * y, npk * 16u);
                bulk_load_u32(S.agst + (uint32_t)(kClAgF + y) * (uint32_t)kClStageBytes, pred_buf + ci.i0, npk * 16u,
                              S.loaded + 8u * y);
            }
            __syncwarp();
            ++m_iss;
            ring_cursor_next(ci, r, n, cb, SP, TP);
            next_pull(ci);
        }
        if (cs.done) break;
        if (m_sto == m_iss) {
            // nothing loaded: publish what is stored, then wait for the predecessor
            if (lane == 0) bulk_wait_all();
            __syncwarp();
            publish(m_sto);
            if (t0 == 0) t0 = globaltimer();
            if ((++spins & 255) == 0 && (globaltimer() - t0 > P.timeout_ns || *(volatile int*)P.err)) {
                if (lane == 0 && !*(volatile int*)P.err) raise_error(P, POLAR_ETIMEOUT);
                ok = false;
            }
            continue;
        }
        t0 = 0;
        // ---- store the oldest loaded tile
        const uint32_t y = m_sto % A;
        if (!__all_sync(0xffffffffu, cl_wait(P, S.loaded + 8u * y, (ldpar >> y) & 1u))) break;
        ldpar ^= 1u << y;
        if (lane == 0) {
            bulk_store_u32(mine + cs.i0, S.agst + (uint32_t)(kClAgF + y) * (uint32_t)kClStageBytes,
                           ring_cursor_npk(cs, TP) * 16u);
            bulk_commit();
        }
        __syncwarp();
        ++m_sto;
        ring_cursor_next(cs, r, n, cb, SP, TP);
        next_pull(cs);
        // ---- publish the tiles whose stores completed (all but the LAG newest)
        if (m_sto > (uint32_t)LAG) {
            if (lane == 0) bulk_wait_group<LAG>();
            __syncwarp();
            publish(m_sto - LAG);
        }
    }
    // the final publication covers every tile, the last final tiles included
    if (lane == 0) bulk_wait_all();
    __syncwarp();
    if (ok) {
        const unsigned long long tw = globaltimer();
        for (;;) {
            publish(m_sto);
            if (pub.q.done) break;
            if (globaltimer() - tw > P.timeout_ns) {
                if (lane == 0) raise_error(P, POLAR_ETIMEOUT);
                break;
            }
        }
    }
}


template <int DT, int OP>
__global__ void __launch_bounds__(kClThreads, POLAR_CL_MINB) ring_cluster_kernel(Params P) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    constexpr int AW = AccWords<DT>::N;
    constexpr int ES = DType<DT>::ES;
    constexpr unsigned TP = cl_tile<AW>();
    const int n = P.nranks;
    const int r = (int)cluster_rank();
    const int c = (int)blockIdx.x / n;
    const int warp = (int)(threadIdx.x >> 5), lane = (int)(threadIdx.x & 31);
    const bool tel = P.tel != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
    const unsigned long long tel_t0 = tel ? globaltimer() : 0;
    extern __shared__ __align__(128) unsigned char smem[];
    const ClRingSmem S = cl_ring_smem(smem_u32(smem));
    const unsigned long long SP = cl_ring_sp<AW>(P);
    unsigned long long ca, cb;
    split_range(0, npacks<ES>(P), P.nch, c, ca, cb);
    char* mine = P.bufs[r];
    // bytes of a received tile: the predecessor sent AW words per pack before its
    // final step (s - 1 < n - 1), one word after
    auto recv_bytes = [&](const RingCursor& q) {
        return ring_cursor_npk(q, TP) * 16u * (uint32_t)(q.s <= n - 1 ? AW : 1);
    };
    if (threadIdx.x == 0) {
        for (int x = 0; x < kClStages; ++x) {
            mbar_init_u32(S.full + 8u * x, 1 + kClWarps);   // the signal warp's expect_tx + every sender warp
            mbar_init_u32(S.cons + 8u * x, kClWarps);
            mbar_init_u32(S.empty + 8u * x, 1);
        }
        for (int x = 0; x < kClOwn; ++x) {
            mbar_init_u32(S.ofull + 8u * x, 1);
            mbar_init_u32(S.oempty + 8u * x, kClWarps);
        }
        for (int x = 0; x < kClAgF; ++x) mbar_init_u32(S.finfull + 8u * x, kClWarps);
        for (int x = 0; x < kClAgP; ++x) mbar_init_u32(S.loaded + 8u * x, 1);
        if (kClAgL2)
            asm volatile("st.shared.u32 [%0], 0;\n\tst.shared.u32 [%1], %3;\n\tst.shared.u32 [%2], 0;" ::"r"(S.cnt),
                         "r"(S.finok), "r"(S.findone), "n"(kClAgF)
                         : "memory");
        mbar_init_u32(S.fin, (uint32_t)(n - 1));
        mbar_fence_init();
        // arm the first kClStages received tiles
        RingCursor q = ring_cursor(r, n, ca, cb, SP);
        for (int x = 0; x < kClStages; ++x) {
            ring_cursor_recv(q, r, n, cb, SP, TP);
            if (q.done) break;
            mbar_expect_u32(S.full + 8u * x, recv_bytes(q));
            ring_cursor_next(q, r, n, cb, SP, TP);
        }
    }
    cluster_sync_all();   // every peer's barriers are initialised before any remote arrive / st.async

    if (warp == 0) {
        // ------------------------------------------------------------- loader
        // own input tiles of the reduce-scatter steps (s <= n-1), in walk order.
        // The whole warp walks (lane 0 issues): a lone lane looping while its
        // warp-mates wait at the final __syncthreads diverges an aligned barrier
        // (measured: the loader starves, 32 MiB takes 65 ms).
        unsigned long long t = 0;
        // POLAR_CL_PF > 0: L2 prefetch of the own tiles that many tiles ahead of
        // the TMA loads (cp.async.bulk.prefetch.L2), so a stage refill hits L2
        RingCursor pf = ring_cursor(r, n, ca, cb, SP);
        unsigned long long npf = 0;
        const bool ok = cl_ring_walk(r, n, ca, cb, SP, TP, [&](int s, unsigned long long i0, unsigned npk) {
            if (s > n - 1) return true;
            const uint32_t x = (uint32_t)(t % kClOwn);
            if (t >= (unsigned long long)kClOwn &&
                !__all_sync(0xffffffffu, cl_wait(P, S.oempty + 8u * x, (uint32_t)((t / kClOwn - 1) & 1))))
                return false;
            if (lane == 0) {
                mbar_expect_u32(S.ofull + 8u * x, npk * 16u);
                bulk_load_u32(S.own + x * (uint32_t)kClStageBytes, mine + i0 * 16ull, npk * 16u, S.ofull + 8u * x);
            }
            ++t;
            if constexpr (kClPf > 0) {
                while (npf < t + (unsigned long long)kClPf) {
                    while (!pf.done && pf.s > n - 1) ring_cursor_next(pf, r, n, cb, SP, TP);
                    if (pf.done) break;
                    if (lane == 0 && npf >= t)
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(mine + pf.i0 * 16ull),
                                     "r"(ring_cursor_npk(pf, TP) * 16u)
                                     : "memory");
                    ring_cursor_next(pf, r, n, cb, SP, TP);
                    ++npf;
                }
            }
            __syncwarp();
            return true;
        });
        if (!ok && lane == 0) {
            // every bulk load issued must land before this CTA's shared memory goes away
            const unsigned long long lo = t > (unsigned long long)kClOwn ? t - kClOwn : 0;
            for (unsigned long long u = lo; u < t; ++u)
                while (!cl_try_wait(S.ofull + 8u * (uint32_t)(u % kClOwn), (uint32_t)((u / kClOwn) & 1))) {}
        }
        __syncwarp();
    } else if (warp == 1) {
        // ------------------------------------------------------------- signal
        // per received tile, once my compute warps have read its stage: re-arm the
        // stage's `full` for the tile kClStages later, then return the credit
        const uint32_t pred = (uint32_t)((r + n - 1) % n);
        const uint32_t pred_empty = cl_map(S.empty, pred);
        RingCursor ahead = ring_cursor(r, n, ca, cb, SP);
        for (int x = 0; x < kClStages && !ahead.done; ++x) {
            ring_cursor_recv(ahead, r, n, cb, SP, TP);
            if (!ahead.done) ring_cursor_next(ahead, r, n, cb, SP, TP);
        }
        unsigned long long nr = 0;
        for (RingCursor q = ring_cursor(r, n, ca, cb, SP);;) {
            ring_cursor_recv(q, r, n, cb, SP, TP);
            if (q.done) break;
            const uint32_t x = (uint32_t)(nr % kClStages);
            if (!__all_sync(0xffffffffu, cl_wait(P, S.cons + 8u * x, (uint32_t)((nr / kClStages) & 1)))) break;
            ring_cursor_recv(ahead, r, n, cb, SP, TP);
            if (lane == 0) {
                if (!ahead.done) mbar_expect_u32(S.full + 8u * x, recv_bytes(ahead));
                cl_arrive_remote(pred_empty + 8u * x);
            }
            __syncwarp();
            if (!ahead.done) ring_cursor_next(ahead, r, n, cb, SP, TP);
            ring_cursor_next(q, r, n, cb, SP, TP);
            ++nr;
        }
    } else if (warp < 2 + kClWarps) {
        // ------------------------------------------------------- compute warps
        const uint32_t succ = (uint32_t)((r + 1) % n);
        ClCompute<DT, OP> cp;
        cp.S = S;
        cp.dst_inbox = cl_map(S.inbox, succ);
        cp.dst_full = cl_map(S.full, succ);
        cp.mine = reinterpret_cast<uint4*>(mine);
        cp.me = (uint32_t)(warp - 2) * 32u + (uint32_t)lane;
        const unsigned long long LC = SP * (unsigned long long)n;
        bool ok = true;
        for (unsigned long long base = ca; base < cb && ok; base += LC) {
            const unsigned long long L = (cb - base < LC) ? cb - base : LC;
            // (all-gather through L2: the compute warps run the reduce-scatter steps only)
            for (int s = 0; s < (kClAgL2 ? n : 2 * (n - 1) + 1) && ok; ++s) {
                int k;
                if (s < n) k = ((r - s) % n + n) % n;
                else k = ((r - (s - n)) % n + n) % n;
                if (s == n - 1) k = (r + 1) % n;
                const unsigned long long ks = base + L * (unsigned long long)k / n;
                const unsigned long long ke = base + L * (unsigned long long)(k + 1) / n;
                // the step's kind is uniform: one specialised tile loop per kind
                if (s == 0) ok = cp.template tiles<kClFirst>(P, ks, ke);
                else if (s < n - 1) ok = cp.template tiles<kClMid>(P, ks, ke);
                else if (s == n - 1) ok = cp.template tiles<kClFin>(P, ks, ke);
                else if (s < 2 * (n - 1)) ok = cp.template tiles<kClAgStep>(P, ks, ke);
                else ok = cp.template tiles<kClLast>(P, ks, ke);
            }
        }
    } else if (warp == 2 + kClWarps) {
        // ------------------------------------------- final-tile store warp (L2)
        cl_ring_fin_warp<AW>(P, S, r, n, ca, cb, SP, reinterpret_cast<uint4*>(mine), lane);
    } else {
        // ------------------------------------------------- all-gather pull warp (L2)
        cl_ring_pull_warp<AW>(P, S, r, n, ca, cb, SP, reinterpret_cast<uint4*>(mine),
                              reinterpret_cast<const uint4*>(P.bufs[(r + n - 1) % n]),
                              cl_map(S.cnt, (uint32_t)((r + 1) % n)), lane);
    }
    cl_rendezvous(P, S.fin, r, n);
    if (tel) {
        volatile TelEntry* e = P.tel + (P.seq % kTelRing);
        e->t0 = tel_t0;
        e->t1 = globaltimer();
        __threadfence_system();
        e->seq = P.seq;
    }
}

// ======================================================================= tree
// Binary tree Simple over a cluster (the FIFO tree's topology and reduction
// order: positions pos = (rank - c) mod n, root = rank c mod n, children
// 2pos+1, 2pos+2; node = own (op) child0 (op) child1, bf16 partials in f32).
// Every hop is an st.async into the receiver's shared-memory inbox; the tree
// is acyclic, so a few stages per link cover the credit round trip.
//   warp 0      loader: own input tiles (TMA) into kTrOwn stages
//   warps 1-4   up group: own (op) children -> parent's up inbox (AW words);
//               the root rounds once, stores, and sends the result down
//   warps 5-8   down group (non-root): parent's result -> HBM + children
// Full barriers are armed by the senders' warps (remote arrive.expect_tx with
// the bytes each warp sent), credits are returned by each consuming warp: the
// up and down groups have kTrGroup warps each, so every count is kTrGroup.
// (With the down phase on DSMEM a double binary tree was slower — interleaved
// tile by tile in one pipeline every tile chains through both trees, 5990 us;
// two concurrent pipelines 1184-2774 us vs 1107 us; profiles/r02dd_*, r02ee_*.
// With the L2 down phase it wins: POLAR_TR_DBT2 below.)
#ifndef POLAR_TR_L2DN
#define POLAR_TR_L2DN 1
#endif
#ifndef POLAR_TR_DBT2
#define POLAR_TR_DBT2 1
#endif
// Defaults per shape (8 x 128 MiB f32, fraction of the HBM copy peak):
//   single tree, L2 down: 16 KiB tiles, up group 4 / 8 / 16 / 24 warps:
//                         0.34 / 0.52 / 0.56 / 0.54
//   double tree (DBT2):   8 KiB tiles, per tree 6 / 8 / 12 up warps:
//                         0.54 / 0.65 / 0.61 (profiles/r02ee_*, r02kk_*)
#if POLAR_TR_DBT2 && POLAR_TR_L2DN
// stages per tree (8 KiB each, 14 fit per tree): up 4 / down 2 / own 4 —
// 8 x 128 MiB f32 499 us, bf16 874 us; up 3 / down 4 / own 4 507 / 885;
// 4/3/3 507 / 898; 5/2/2 551 / 895; 4/4/2 555 / 913 (profiles/r02pp_*)
#define POLAR_TR_WIRE_D 512
#define POLAR_TR_UP_D 4
#define POLAR_TR_DN_D 2
#define POLAR_TR_OWN_D 4
#define POLAR_TR_GROUP_D 8
#elif POLAR_TR_L2DN
#define POLAR_TR_WIRE_D 1024
#define POLAR_TR_UP_D 4
#define POLAR_TR_DN_D 3
#define POLAR_TR_OWN_D 2
#define POLAR_TR_GROUP_D 16
#else
#define POLAR_TR_WIRE_D 1024
#define POLAR_TR_UP_D 4
#define POLAR_TR_DN_D 3
#define POLAR_TR_OWN_D 2
#define POLAR_TR_GROUP_D 4
#endif
#ifndef POLAR_TR_WIRE
#define POLAR_TR_WIRE POLAR_TR_WIRE_D   // 16-B wire words per stage
#endif
#ifndef POLAR_TR_UP
#define POLAR_TR_UP POLAR_TR_UP_D       // stages per child up inbox
#endif
#ifndef POLAR_TR_DN
#define POLAR_TR_DN POLAR_TR_DN_D       // down stages (pull / staging in L2 mode)
#endif
#ifndef POLAR_TR_OWN
#define POLAR_TR_OWN POLAR_TR_OWN_D     // own-input stages
#endif
#ifndef POLAR_TR_GROUP
#define POLAR_TR_GROUP POLAR_TR_GROUP_D // up-group warps (per tree)
#endif
// POLAR_TR_L2DN (the default): the down phase through L2 instead of DSMEM.  The
// root's up group stages each result tile in shared memory; one down warp
// bulk-stores it into the root's buffer and, once the store has completed,
// publishes the count of tiles in that buffer to each child (relaxed remote
// store); a non-root's down warp pulls its parent's published tiles from the
// parent's buffer with TMA loads and bulk-stores them into its own, publishing
// in turn.  DSMEM then carries only the up phase: an interior node moves 2
// tiles in and 1 out per tile (f32) instead of 3 and 3.
constexpr bool kTrL2 = POLAR_TR_L2DN != 0;
// POLAR_TR_DBT2 (the default, with the L2 down phase): a double binary tree —
// the channel's tiles cut in halves, the second half through the tree with
// every position shifted by ceil(n/2) (its interior nodes are the first
// tree's leaves); the two trees run concurrently on disjoint warps and shared
// memory.  With the down phase in L2 a leaf receives nothing through DSMEM, so
// no SM takes in more than 2 tiles per 2 tiles of the channel instead of 2 per
// tile.  (The reduction order of the second half differs from the FIFO
// tree's: f32 sums match it within the tree's bound, integer-valued exactly.)
constexpr int kTrTrees = (POLAR_TR_DBT2 && POLAR_TR_L2DN) ? 2 : 1;
constexpr unsigned kTrWire = POLAR_TR_WIRE;
constexpr size_t kTrStage = (size_t)kTrWire * 16;
constexpr int kTrUp = POLAR_TR_UP, kTrDn = POLAR_TR_DN, kTrOwn = POLAR_TR_OWN, kTrGroup = POLAR_TR_GROUP;
constexpr int kTrWarpsPerTree = 1 + kTrGroup + (kTrL2 ? 1 : kTrGroup);
constexpr int kTrThreads = 32 * kTrWarpsPerTree * kTrTrees;
constexpr int kTrNbar = 2 * kTrUp + kTrUp + kTrDn + 2 * kTrDn + 2 * kTrOwn + 1;
// one tree's shared memory, padded to 128 B so that the second tree's stages
// stay 128-B aligned (bulk copies and 16-B st.async need >= 16 B; an odd
// barrier count left them 8-B aligned: cudaErrorMisalignedAddress)
__host__ __device__ constexpr size_t cl_tree_bytes_per_tree() {
    return ((size_t)(2 * kTrUp + kTrDn + kTrOwn) * kTrStage + (size_t)kTrNbar * 8 + 16 + 127) & ~(size_t)127;
}
__host__ __device__ constexpr size_t cl_tree_smem_bytes() { return cl_tree_bytes_per_tree() * kTrTrees; }
static_assert(kTrStage % 128 == 0, "tree stages must keep 128-B alignment");
struct ClTreeSmem {
    uint32_t up[2], dn, own;            // inboxes (child k up, parent down), own stages
    uint32_t upfull[2], upempty;        // up inbox k landed / my up sends' credits
    uint32_t dnfull, dnempty[2];        // down inbox landed / my down sends to child k: credits
    uint32_t ofull, oempty, fin;
    uint32_t cnt, stok;                 // L2 down: parent's published tiles; root staging stages handed out
};
__device__ __forceinline__ ClTreeSmem cl_tree_smem(uint32_t base) {
    ClTreeSmem t;
    uint32_t o = base;
    t.up[0] = o; o += (uint32_t)(kTrUp * kTrStage);
    t.up[1] = o; o += (uint32_t)(kTrUp * kTrStage);
    t.dn = o; o += (uint32_t)(kTrDn * kTrStage);
    t.own = o; o += (uint32_t)(kTrOwn * kTrStage);
    t.upfull[0] = o; o += 8u * kTrUp;
    t.upfull[1] = o; o += 8u * kTrUp;
    t.upempty = o; o += 8u * kTrUp;
    t.dnfull = o; o += 8u * kTrDn;
    t.dnempty[0] = o; o += 8u * kTrDn;
    t.dnempty[1] = o; o += 8u * kTrDn;
    t.ofull = o; o += 8u * kTrOwn;
    t.oempty = o; o += 8u * kTrOwn;
    t.fin = o;
    t.cnt = o + 8u;
    t.stok = o + 12u;
    return t;
}
// a ring counter: stage index and the parity of the phase to wait for
struct StageCtr {
    uint32_t x = 0, par = 0;
    bool wrapped = false;
    __device__ __forceinline__ void next(uint32_t D) {
        if (++x == D) { x = 0; par ^= 1u; wrapped = true; }
    }
};

// The L2 down phase (POLAR_TR_L2DN), one warp, lane 0 drives:
//   root     result tiles staged by the up group -> bulk store into my buffer
//   non-root my parent's published tiles -> TMA load into a stage -> bulk store
//            into my buffer
// then, once a tile's store has completed (bulk group), publish "tiles in my
// buffer" to each child (relaxed remote store: the completed group is what
// orders the data; a cluster-scope release costs ~75 us here, §8).  Stages:
// kTrDn; the root hands a staging stage back (stok) once its store has read it.
template <int AW>
__device__ __noinline__ void tree_down_l2(const Params& P, const ClTreeSmem S, bool root, int nchild,
                                          const uint32_t (&ch_cnt)[2], const uint4* par_buf, uint4* mine,
                                          unsigned long long ca, unsigned long long cb, int lane) {
    constexpr unsigned TP = kTrWire / (unsigned)AW;
    constexpr int D = kTrDn;
    const uint32_t ntiles = (uint32_t)((cb - ca + TP - 1) / TP);
    uint32_t t_iss = 0, t_sto = 0, seen = 0, published = 0, par = 0;
    unsigned long long t0 = 0;
    uint32_t spins = 0;
    bool ok = true;
    auto publish = [&](uint32_t done) {
        if (done != published) {
            if (lane == 0)
                for (int k = 0; k < nchild; ++k) cl_st_release_remote_u32(ch_cnt[k], done);
            published = done;
        }
        __syncwarp();
    };
    while (ok && t_sto < ntiles) {
        if (!root) {
            // issue loads ahead, as the parent's count allows
            while (t_iss < ntiles && t_iss < t_sto + D) {
                if (seen < t_iss + 1) {
                    uint32_t v = 0;
                    if (lane == 0) v = cl_ld_acquire_u32(S.cnt);
                    seen = __shfl_sync(0xffffffffu, v, 0);
                    if (seen < t_iss + 1) break;
                }
                const uint32_t x = t_iss % D;
                const unsigned long long i0 = ca + (unsigned long long)t_iss * TP;
                const unsigned npk = (unsigned)((cb - i0) < TP ? (cb - i0) : TP);
                if (lane == 0) {
                    if (t_iss >= (uint32_t)D) bulk_wait_read<0>();   // the stage's previous store has read it
                    mbar_expect_u32(S.dnfull + 8u * x, npk * 16u);
                    bulk_load_u32(S.dn + x * (uint32_t)kTrStage, par_buf + i0, npk * 16u, S.dnfull + 8u * x);
                }
                __syncwarp();
                ++t_iss;
            }
            if (t_sto == t_iss) {
                // nothing loaded: publish what is stored, then wait for the parent
                if (lane == 0) bulk_wait_all();
                __syncwarp();
                publish(t_sto);
                if (t0 == 0) t0 = globaltimer();
                if ((++spins & 255) == 0 && (globaltimer() - t0 > P.timeout_ns || *(volatile int*)P.err)) {
                    if (lane == 0 && !*(volatile int*)P.err) raise_error(P, POLAR_ETIMEOUT);
                    ok = false;
                }
                continue;
            }
            t0 = 0;
        }
        // store the oldest ready tile
        const uint32_t x = t_sto % D;
        {
            int rd = 0;
            if (lane == 0) rd = cl_try_wait(S.dnfull + 8u * x, (par >> x) & 1u);
            rd = __shfl_sync(0xffffffffu, rd, 0);
            if (!rd) {   // about to block: publish what is stored first
                if (lane == 0) bulk_wait_all();
                __syncwarp();
                publish(t_sto);
            }
        }
        if (!__all_sync(0xffffffffu, cl_wait(P, S.dnfull + 8u * x, (par >> x) & 1u))) break;
        par ^= 1u << x;
        const unsigned long long i0 = ca + (unsigned long long)t_sto * TP;
        const unsigned npk = (unsigned)((cb - i0) < TP ? (cb - i0) : TP);
        if (lane == 0) {
            bulk_store_u32(mine + i0, S.dn + x * (uint32_t)kTrStage, npk * 16u);
            bulk_commit();
            if (root) {
                bulk_wait_read<0>();   // hand the staging stage back to the up group
                asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(S.stok), "r"(t_sto + 1 + D) : "memory");
            }
            bulk_wait_group<1>();      // all but this store have completed
        }
        __syncwarp();
        publish(t_sto);
        ++t_sto;
    }
    if (lane == 0) bulk_wait_all();
    __syncwarp();
    if (ok) publish(t_sto);
}

template <int DT, int OP>
__global__ void __launch_bounds__(kTrThreads, 1) tree_cluster_kernel(Params P) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    constexpr int AW = AccWords<DT>::N;
    constexpr int ES = DType<DT>::ES;
    constexpr unsigned TP = kTrWire / (unsigned)AW;            // element packs per tile
    constexpr unsigned NT = kTrGroup * 32;
    constexpr unsigned PPL = (TP + NT - 1) / NT;
    const int n = P.nranks;
    const int r = (int)cluster_rank();
    const int c = (int)blockIdx.x / n;
    const int lane = (int)(threadIdx.x & 31);
    const int tree = (int)(threadIdx.x >> 5) / kTrWarpsPerTree;            // (POLAR_TR_DBT2: 0 or 1)
    const int warp = (int)(threadIdx.x >> 5) % kTrWarpsPerTree;            // role within the tree
    const int shift = tree * ((n + 1) / 2);
    const int pos = ((r - c + shift) % n + n) % n;
    auto rank_of = [&](int q) { return ((q - shift + c) % n + n) % n; };
    const bool root = pos == 0;
    const int parent = root ? -1 : rank_of((pos - 1) / 2);
    const int my_idx = root ? 0 : (pos - 1) % 2;
    int child[2] = {-1, -1};
    int nchild = 0;
    for (int k = 0; k < 2; ++k)
        if (2 * pos + 1 + k < n) { child[k] = rank_of(2 * pos + 1 + k); nchild = k + 1; }
    const bool tel = P.tel != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
    const unsigned long long tel_t0 = tel ? globaltimer() : 0;
    extern __shared__ __align__(128) unsigned char smem[];
    const ClTreeSmem S = cl_tree_smem(smem_u32(smem) + (uint32_t)(tree * cl_tree_bytes_per_tree()));
    const uint32_t fin0 = cl_tree_smem(smem_u32(smem)).fin;   // the CTA's rendezvous (tree 0's)
    if (warp == 0 && lane == 0) {
        for (int x = 0; x < kTrUp; ++x) {
            mbar_init_u32(S.upfull[0] + 8u * x, kTrGroup);
            mbar_init_u32(S.upfull[1] + 8u * x, kTrGroup);
            mbar_init_u32(S.upempty + 8u * x, kTrGroup);
        }
        for (int x = 0; x < kTrDn; ++x) {
            // L2 down: the root's staging stages are filled by its up group, a
            // non-root's pull stages by one TMA load each
            mbar_init_u32(S.dnfull + 8u * x, (kTrL2 && !root) ? 1u : (uint32_t)kTrGroup);
            mbar_init_u32(S.dnempty[0] + 8u * x, kTrGroup);
            mbar_init_u32(S.dnempty[1] + 8u * x, kTrGroup);
        }
        for (int x = 0; x < kTrOwn; ++x) {
            mbar_init_u32(S.ofull + 8u * x, 1);
            mbar_init_u32(S.oempty + 8u * x, kTrGroup);
        }
        if (kTrL2)
            asm volatile("st.shared.u32 [%0], 0;\n\tst.shared.u32 [%1], %2;" ::"r"(S.cnt), "r"(S.stok), "n"(kTrDn)
                         : "memory");
        if (tree == 0) mbar_init_u32(S.fin, (uint32_t)(n - 1));
        mbar_fence_init();
    }
    cluster_sync_all();
    unsigned long long ca, cb;
    split_range(0, npacks<ES>(P), P.nch, c, ca, cb);
    if (kTrTrees > 1) {
        // tree t takes half of the channel's tiles
        const unsigned long long tiles = (cb - ca + TP - 1) / TP;
        const unsigned long long mid = ca + (tiles + 1) / 2 * TP < cb ? ca + (tiles + 1) / 2 * TP : cb;
        if (tree == 0) cb = mid;
        else ca = mid;
    }
    uint4* mine = reinterpret_cast<uint4*>(P.bufs[r]);
    // remote addresses: my up inbox slot at the parent, the children's down inboxes
    const uint32_t par_up = root ? 0u : cl_map(S.up[my_idx], (uint32_t)parent);
    const uint32_t par_upfull = root ? 0u : cl_map(S.upfull[my_idx], (uint32_t)parent);
    const uint32_t par_dnempty = root ? 0u : cl_map(S.dnempty[my_idx], (uint32_t)parent);
    uint32_t ch_dn[2] = {0, 0}, ch_dnfull[2] = {0, 0}, ch_upempty[2] = {0, 0};
    for (int k = 0; k < nchild; ++k) {
        ch_dn[k] = cl_map(S.dn, (uint32_t)child[k]);
        ch_dnfull[k] = cl_map(S.dnfull, (uint32_t)child[k]);
        ch_upempty[k] = cl_map(S.upempty, (uint32_t)child[k]);
    }
    // the bytes a warp of a group sends for its packs of a tile of npk packs
    auto warp_packs = [&](int gw, unsigned npk) {
        uint32_t cnt = 0;
#pragma unroll
        for (unsigned u = 0; u < PPL; ++u) {
            const unsigned b0 = u * NT + (unsigned)gw * 32;
            cnt += npk > b0 ? (npk - b0 < 32 ? npk - b0 : 32) : 0;
        }
        return cnt;
    };

    if (warp == 0) {
        // ------------------------------------------------------------- loader
        StageCtr w;
        bool ok = true;
        unsigned long long issued = 0;
        for (unsigned long long i0 = ca; i0 < cb && ok; i0 += TP) {
            const unsigned npk = (unsigned)((cb - i0) < TP ? (cb - i0) : TP);
            if (w.wrapped && !__all_sync(0xffffffffu, cl_wait(P, S.oempty + 8u * w.x, w.par ^ 1u))) { ok = false; break; }
            if (lane == 0) {
                mbar_expect_u32(S.ofull + 8u * w.x, npk * 16u);
                bulk_load_u32(S.own + w.x * (uint32_t)kTrStage, mine + i0, npk * 16u, S.ofull + 8u * w.x);
            }
            __syncwarp();
            ++issued;
            w.next(kTrOwn);
        }
        if (!ok && lane == 0) {
            const unsigned long long lo = issued > (unsigned long long)kTrOwn ? issued - kTrOwn : 0;
            for (unsigned long long u = lo; u < issued; ++u)
                while (!cl_try_wait(S.ofull + 8u * (uint32_t)(u % kTrOwn), (uint32_t)((u / kTrOwn) & 1))) {}
        }
        __syncwarp();
    } else if (warp <= kTrGroup) {
        // ----------------------------------------------------------- up group
        const int gw = warp - 1;
        const unsigned me = (unsigned)gw * 32u + (unsigned)lane;
        StageCtr w, in, up, dn;   // own stage, child up inboxes (both children in step), my up sends, my down sends
        uint32_t jt = 0;          // tiles done
        for (unsigned long long i0 = ca; i0 < cb; i0 += TP) {
            const unsigned npk = (unsigned)((cb - i0) < TP ? (cb - i0) : TP);
            if (!cl_wait(P, S.ofull + 8u * w.x, w.par)) break;
            bool ok = true;
            for (int k = 0; k < nchild; ++k) ok = ok && cl_wait(P, S.upfull[k] + 8u * in.x, in.par);
            if (!root && up.wrapped) ok = ok && cl_wait(P, S.upempty + 8u * up.x, up.par ^ 1u);
            if (root && !kTrL2)
                for (int k = 0; k < nchild; ++k)
                    if (dn.wrapped) ok = ok && cl_wait(P, S.dnempty[k] + 8u * dn.x, dn.par ^ 1u);
            // L2 down: the root stages its result tile for the down warp (a
            // monotone hand-out count, no parity to alias)
            if (root && kTrL2) ok = ok && cl_wait_count(P, S.stok, jt + 1);
            if (!ok) break;
            const uint32_t stg = S.dn + (uint32_t)(jt % kTrDn) * (uint32_t)kTrStage;
            const uint32_t ow = S.own + w.x * (uint32_t)kTrStage;
            const uint32_t cin0 = S.up[0] + in.x * (uint32_t)kTrStage, cin1 = S.up[1] + in.x * (uint32_t)kTrStage;
            const uint32_t dst = par_up + up.x * (uint32_t)kTrStage, dbar = par_upfull + 8u * up.x;
            if (!root || nchild) jitter_warp(P);
#pragma unroll
            for (unsigned u = 0; u < PPL; ++u) {
                const unsigned p = u * NT + me;
                if (p >= npk) break;
                Acc<DT> acc;
                acc_init<DT>(acc, ld_shared_v4(ow + p * 16u));
                for (int k = 0; k < nchild; ++k) {
                    Acc<DT> chv;
#pragma unroll
                    for (int q = 0; q < AW; ++q) chv.w[q] = ld_shared_v4((k ? cin1 : cin0) + ((unsigned)q * TP + p) * 16u);
                    acc_merge<DT, OP>(acc, chv);
                }
                if (root && kTrL2) {
                    const uint4 v = acc_fin<DT>(acc);
                    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(stg + p * 16u), "r"(v.x), "r"(v.y),
                                 "r"(v.z), "r"(v.w)
                                 : "memory");
                } else if (root) {
                    const uint4 v = acc_fin<DT>(acc);
                    st_plain(mine + i0 + p, v);
                    for (int k = 0; k < nchild; ++k) cl_st_async(ch_dn[k] + dn.x * (uint32_t)kTrStage + p * 16u, v,
                                                                 ch_dnfull[k] + 8u * dn.x);
                } else {
#pragma unroll
                    for (int q = 0; q < AW; ++q) cl_st_async(dst + ((unsigned)q * TP + p) * 16u, acc.w[q], dbar);
                }
            }
            if (root && kTrL2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // -> the bulk store
            __syncwarp();
            if (lane == 0) {
                const uint32_t cnt = warp_packs(gw, npk);
                mbar_arrive_u32(S.oempty + 8u * w.x);
                for (int k = 0; k < nchild; ++k) cl_arrive_remote(ch_upempty[k] + 8u * in.x);   // credits to children
                if (!root) cl_arrive_expect_remote(dbar, cnt * 16u * (uint32_t)AW);
                else if (kTrL2) mbar_arrive_rel_u32(S.dnfull + 8u * (jt % kTrDn));
                else
                    for (int k = 0; k < nchild; ++k) cl_arrive_expect_remote(ch_dnfull[k] + 8u * dn.x, cnt * 16u);
            }
            ++jt;
            w.next(kTrOwn);
            if (nchild) in.next(kTrUp);
            if (!root) up.next(kTrUp);
            else if (nchild) dn.next(kTrDn);
        }
    } else if (kTrL2) {
        // ------------------------------------------------ down warp (L2 down)
        if (warp == 1 + kTrGroup) {
            uint32_t ch_cnt[2] = {0, 0};
            for (int k = 0; k < nchild; ++k) ch_cnt[k] = cl_map(S.cnt, (uint32_t)child[k]);
            tree_down_l2<AW>(P, S, root, nchild, ch_cnt, root ? nullptr : reinterpret_cast<const uint4*>(P.bufs[parent]),
                             mine, ca, cb, lane);
        }
    } else if (!root) {
        // --------------------------------------------------------- down group
        const int gw = warp - 1 - kTrGroup;
        const unsigned me = (unsigned)gw * 32u + (unsigned)lane;
        StageCtr in, dn;
        for (unsigned long long i0 = ca; i0 < cb; i0 += TP) {
            const unsigned npk = (unsigned)((cb - i0) < TP ? (cb - i0) : TP);
            bool ok = cl_wait(P, S.dnfull + 8u * in.x, in.par);
            for (int k = 0; k < nchild; ++k)
                if (dn.wrapped) ok = ok && cl_wait(P, S.dnempty[k] + 8u * dn.x, dn.par ^ 1u);
            if (!ok) break;
            const uint32_t src = S.dn + in.x * (uint32_t)kTrStage;
            if (nchild) jitter_warp(P);
#pragma unroll
            for (unsigned u = 0; u < PPL; ++u) {   // down tiles: TP packs of one word
                const unsigned p = u * NT + me;
                if (p >= npk) break;
                const uint4 v = ld_shared_v4(src + p * 16u);
                st_plain(mine + i0 + p, v);
                for (int k = 0; k < nchild; ++k) cl_st_async(ch_dn[k] + dn.x * (uint32_t)kTrStage + p * 16u, v,
                                                             ch_dnfull[k] + 8u * dn.x);
            }
            __syncwarp();
            if (lane == 0) {
                const uint32_t cnt = warp_packs(gw, npk);
                cl_arrive_remote(par_dnempty + 8u * in.x);   // credit to the parent
                for (int k = 0; k < nchild; ++k) cl_arrive_expect_remote(ch_dnfull[k] + 8u * dn.x, cnt * 16u);
            }
            in.next(kTrDn);
            if (nchild) dn.next(kTrDn);
        }
    }
    cl_rendezvous(P, fin0, r, n);
    if (tel) {
        volatile TelEntry* e = P.tel + (P.seq % kTelRing);
        e->t0 = tel_t0;
        e->t1 = globaltimer();
        __threadfence_system();
        e->seq = P.seq;
    }
}

}  // namespace dev
}  // namespace polar
