// The AllReduce kernels.
//
// One kernel per <dtype, op, algorithm, protocol>.  Grid = nlocal x nch CTAs:
// block b serves rank rank0 + b / nch on channel c = b % nch (a real comm has
// nlocal = 1; a virtual comm hosts every rank in one cooperative launch).
// Every cross-rank exchange is a direct load/store on a peer-mapped pointer
// (NVLink/NVSwitch on a real node), ordered by u64 flags or flag-in-data LL
// lines; nothing goes through NCCL or the host.
//
// Reduction order (R2-R4):
//   one-shot / two-shot : x_0 (op) x_1 (op) ... (op) x_{n-1}   == the oracle, bit for bit
//   ring                : chunk k starts at rank k and follows the ring
//   tree                : node = own (op) child0 (op) child1, root rotated per channel
// bf16 accumulates in f32 everywhere and is rounded once per output element.
#pragma once
#include "device.cuh"

namespace polar {
namespace dev {

struct Who {
    int r, c, n, tid;
};

__device__ __forceinline__ Who who(const Params& P) {
    Who w;
    w.r = P.rank0 + (int)blockIdx.x / P.nch;
    w.c = (int)blockIdx.x % P.nch;
    w.n = P.nranks;
    w.tid = (int)threadIdx.x;
    return w;
}

template <int ES> __device__ __forceinline__ unsigned long long npacks(const Params& P) {
    return (P.count + (16 / ES) - 1) / (16 / ES);
}

// One-shot / two-shot epochs are PER CALL, not per channel: every channel's
// ChanState.epoch holds the same value and each call advances all kMaxCh of
// them (CTA c writes channels c, c+nch, ...).  Staging is shared by all
// channels, so a per-channel epoch could let channel c' see channel c's stale LL
// line carrying the same flag value after the channel count changed.
__device__ __forceinline__ void epoch_publish(const Params& P, const Who& w, uint64_t e) {
    if (w.tid == 0)
        for (int cc = w.c; cc < kMaxCh; cc += P.nch) chan_state(P, w.r, cc)->epoch = e;
}

// Staged (one-shot / two-shot LL) chunk geometry.  Each chunk gives every
// channel a FIXED region of `per` packs inside a staging slot (offset c*per), so
// no two channels ever share a staging location, whatever the chunk (a short
// last chunk must not re-slice: a lagging peer channel may still be polling the
// same-parity slot of two chunks ago).  `per` is the same on every rank and for
// every chunk of a call: min(slot capacity / nch, ceil(NP / (parts*nch))),
// rounded to whole UNITs (32 packs = 512 B; 30 packs = one LL128 warp unit, so
// that channel regions start on a line group).
struct Geo {
    unsigned long long per;      // packs per channel per part per chunk
    unsigned long long part;     // per * nch: packs per part (owner) per chunk
    unsigned long long chunk;    // part * parts
    unsigned long long nchunks;
};
template <unsigned long long UNIT>
__device__ __forceinline__ Geo make_geo(unsigned long long NP, unsigned long long cap_packs, int nch, int parts) {
    Geo g;
    unsigned long long cap = (cap_packs / (unsigned long long)nch) / UNIT * UNIT;
    unsigned long long need = (NP + (unsigned long long)(parts * nch) - 1) / (unsigned long long)(parts * nch);
    need = (need + UNIT - 1) / UNIT * UNIT;
    g.per = need < cap ? need : cap;
    if (g.per < UNIT) g.per = UNIT;
    g.part = g.per * (unsigned long long)nch;
    g.chunk = g.part * (unsigned long long)parts;
    g.nchunks = (NP + g.chunk - 1) / g.chunk;
    return g;
}
// channel c's packs of part j in chunk k: [lo, hi) and the slot offset of lo
__device__ __forceinline__ void geo_slice(const Geo& g, unsigned long long NP, unsigned long long k, int j, int c,
                                          unsigned long long& lo, unsigned long long& hi, unsigned long long& off) {
    off = g.per * (unsigned long long)c;
    lo = k * g.chunk + g.part * (unsigned long long)j + off;
    hi = lo + g.per;
    if (lo > NP) lo = NP;
    if (hi > NP) hi = NP;
}

// Entry / exit handshakes of the zero-copy kernels (two-shot Simple, the direct
// collectives): entry = every rank's input is ready; exit = no peer still reads
// or writes my buffer.  A real comm needs both: its peers are other processes'
// launches.  A virtual comm runs every rank in ONE grid, which starts after the
// inputs' producers (stream order; griddepcontrol.wait under PDL) and whose
// completion precedes any later use of the buffers, and the zero-copy kernels
// have no other cross-rank dependency — so the launch subsumes both handshakes
// and virtual comms skip them (POLAR_VIRTUAL_HANDSHAKE=1 builds keep them).
#ifndef POLAR_VIRTUAL_HANDSHAKE
#define POLAR_VIRTUAL_HANDSHAKE 0
#endif
// The entry handshake also carries the launch's decision tag (F_ENTRY_SIG,
// written before the release of F_ENTRY): a rank whose peers addressed this
// call differently (another registration or offset, the bounce path, another
// count / op / dtype / channel count) sees a foreign tag right after the
// barrier, latches POLAR_ESTATE and leaves before any data moves — every rank
// sees the difference (it is symmetric), so all of them leave and none waits.
__device__ __forceinline__ bool handshake_entry(const Params& P, const Who& w, uint64_t e) {
    if (!P.sys && !POLAR_VIRTUAL_HANDSHAKE) return true;
    if (w.tid < w.n) {
        jitter(P);
        if (P.sys) st_relaxed(flag_ptr(P, w.tid, F_ENTRY_SIG, w.c, w.r), P.dtag, P.sys);
        st_release(flag_ptr(P, w.tid, F_ENTRY, w.c, w.r), e, P.sys);
    }
    bool ok = true;
    if (w.tid < w.n) {
        ok = wait_geq(P, flag_ptr(P, w.r, F_ENTRY, w.c, w.tid), e);
        if (ok && P.sys && *(volatile const uint64_t*)flag_ptr(P, w.r, F_ENTRY_SIG, w.c, w.tid) != P.dtag) {
            raise_error(P, POLAR_ESTATE);
            ok = false;
        }
    }
    return __syncthreads_and(ok) != 0;
}
__device__ __forceinline__ bool handshake_exit(const Params& P, const Who& w, uint64_t e) {
    if (!P.sys && !POLAR_VIRTUAL_HANDSHAKE) return true;
    if (w.tid < w.n) {
        fence_acq_rel(P.sys);
        jitter(P), st_relaxed(flag_ptr(P, w.tid, F_EXIT, w.c, w.r), e, P.sys);
    }
    bool ok = true;
    if (w.tid < w.n) ok = wait_geq(P, flag_ptr(P, w.r, F_EXIT, w.c, w.tid), e);
    return __syncthreads_and(ok) != 0;
}

// ===================================================================== two-shot
// Simple, zero-copy on symmetric buffers: entry barrier; owner r reads shard r
// from every rank, reduces in rank order, stores the result into every rank's
// shard r; exit barrier.  NVLink bytes per rank: 2(n-1)/n * S.

// Dynamic chunk loop of the zero-copy two-shot, specialised on the rank count:
// N in {2,3,4} keeps U = 8/N packs per thread in flight (8 independent 16-B
// loads, so small n does not starve the memory system); N = 0 is the generic
// predicated path (one pack x n ranks; n >= 5 already has >= 5 loads in flight).
// Templating the WHOLE loop (not just its body) keeps each variant's pointers
// out of the others' live ranges (the body-level switch spilled at 128 regs).
struct TwoShotGeo {
    unsigned long long s0, s1, nbig, bigend, nchunks, nfull, wbase;
    unsigned long long big, small;   // chunk sizes in packs
    unsigned long long* work;
};
#ifndef POLAR_TS_BIG
#define POLAR_TS_BIG 1024
#endif
#ifndef POLAR_TS_SMALL
#define POLAR_TS_SMALL 512
#endif
#ifndef POLAR_TS_UGEN
#define POLAR_TS_UGEN 1   // packs per thread per rank in flight on the generic (n >= 5) path
#endif
constexpr unsigned long long kTsBig = POLAR_TS_BIG, kTsSmall = POLAR_TS_SMALL;   // packs (16 KiB / 8 KiB per buffer)
// the TMA pipeline restarts per grab, so it takes bigger chunks (32 KiB per buffer:
// n = 2 at 1 GiB 906 -> 1098 GB/s busBW vs 16 KiB)
constexpr unsigned long long kTsBigTma = 2048;

template <int DT, int OP, int N>
__device__ __forceinline__ void twoshot_loop(const Params& P, const Who& w, const TwoShotGeo& g) {
    constexpr int ES = DType<DT>::ES;
    constexpr int NR = N ? N : kMaxRanks;
    constexpr int U = (N >= 2 && N <= 4) ? 8 / N : POLAR_TS_UGEN;
    const int n = w.n, tid = w.tid;
    __shared__ unsigned long long s_next;
    if (tid == 0) {
        atomicMax(g.work, g.wbase);
        s_next = atomicAdd(g.work, 1ull) - g.wbase;
    }
    __syncthreads();
    unsigned long long k = s_next;
    const uint4* src[NR];
#pragma unroll
    for (int p = 0; p < NR; ++p) src[p] = reinterpret_cast<const uint4*>(P.bufs[(N || p < n) ? p : 0]);
    const unsigned long long stride = (unsigned long long)blockDim.x;
    while (k < g.nchunks) {
        __syncthreads();                                         // everyone has read s_next
        if (tid == 0) s_next = atomicAdd(g.work, 1ull) - g.wbase;   // prefetch the next grab
        const unsigned long long a = g.s0 + (k < g.nbig ? k * g.big : g.bigend + (k - g.nbig) * g.small);
        unsigned long long b = a + (k < g.nbig ? g.big : g.small);
        if (b > g.s1) b = g.s1;
        if (b <= g.nfull) {
            // fast path: full, 16-B aligned packs
#pragma unroll 1
            for (unsigned long long i0 = a + tid; i0 < b; i0 += U * stride) {
                uint4 v[U][NR];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const unsigned long long i = i0 + u * stride;
                    if (i < b) {
#pragma unroll
                        for (int p = 0; p < NR; ++p)
                            if (N || p < n) v[u][p] = ld_cg(src[p] + i);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const unsigned long long i = i0 + u * stride;
                    if (i < b) {
                        Acc<DT> acc;
                        acc_init<DT>(acc, v[u][0]);
#pragma unroll
                        for (int p = 1; p < NR; ++p)
                            if (N || p < n) acc_add<DT, OP>(acc, v[u][p]);
                        const uint4 out = acc_fin<DT>(acc);
#pragma unroll
                        for (int p = 0; p < NR; ++p)
                            if (N || p < n) st_plain(const_cast<uint4*>(src[p]) + i, out);
                    }
                }
            }
        } else {
            // partial last pack / unaligned buffers: element-exact copies
            for (unsigned long long i = a + tid; i < b; i += blockDim.x) {
                Acc<DT> acc;
                acc_init<DT>(acc, load_pack<ES>(P, P.bufs[0], i));
                for (int p = 1; p < n; ++p) acc_add<DT, OP>(acc, load_pack<ES>(P, P.bufs[p], i));
                const uint4 out = acc_fin<DT>(acc);
                for (int p = 0; p < n; ++p) store_pack<ES>(P, P.bufs[p], i, out);
            }
        }
        __syncthreads();                                         // chunk done, s_next visible
        k = s_next;
    }
}


// TMA-staged variant of the zero-copy two-shot loop (Params.tma), warp
// specialised.  Warp 0 / lane 0 is the producer: it grabs chunks from the same
// per-owner counter, cuts them into (32 KiB / n)-per-rank tiles, issues one
// cp.async.bulk load per rank into a shared-memory stage (its `full` mbarrier
// counts the bytes), and once the consumers have released a stage (`empty`
// mbarrier, one arrival per consumer warp) issues one bulk store per rank of
// the reduced tile and reuses the stage after the stores have read it.  Warps
// 1..15 reduce each stage in rank order from shared memory into the rank-0
// slot.  kTmaStages stages of 32 KiB per CTA.  Only full 16-B packs go through
// TMA; the partial last pack (if any) is finished with the slow path.
template <int DT, int OP>
__device__ void twoshot_tma(const Params& P, const Who& w, const TwoShotGeo& g) {
    constexpr int ES = DType<DT>::ES;
    extern __shared__ __align__(128) unsigned char smem[];
    const int n = w.n, tid = w.tid;
    const int warp = tid >> 5, lane = tid & 31;
    const int nconsumer_warps = (int)(blockDim.x >> 5) - 1;
    const unsigned tile_pk = tma_tile_packs(n);             // packs per rank per tile
    const size_t tile_b = (size_t)tile_pk * 16;
    unsigned char* data = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)kTmaStages * kTmaStageBytes);
    uint64_t* empty = full + kTmaStages;
    unsigned long long* meta_off = reinterpret_cast<unsigned long long*>(empty + kTmaStages);
    unsigned long long* meta_npk = meta_off + kTmaStages;
    __shared__ unsigned long long s_tail_lo, s_tail_hi;   // slow-path remainder grabbed by this CTA
    if (tid == 0) {
        for (int st = 0; st < kTmaStages; ++st) {
            mbar_init(&full[st], 1);
            mbar_init(&empty[st], (uint32_t)nconsumer_warps);
        }
        mbar_fence_init();
        s_tail_lo = s_tail_hi = 0;
    }
    __syncthreads();
    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------------- producer
            atomicMax(g.work, g.wbase);
            unsigned long long pos = 0, fend = 0, tail_lo = 0, tail_hi = 0;
            bool done = false;
            // iteration t: drain tile d = t-(S-1) (wait for its reduction, issue its
            // stores), then load tile t into stage t%S, whose previous tile t-S was
            // drained one iteration ago: wait_group.read<1> lets the stores just
            // issued stay in flight while guaranteeing that older ones have read.
            for (unsigned t = 0;; ++t) {
                const int st = (int)(t % kTmaStages);
                if (t >= (unsigned)(kTmaStages - 1)) {
                    const unsigned d = t - (kTmaStages - 1);
                    const int sd = (int)(d % kTmaStages);
                    while (!mbar_try_wait(&empty[sd], (d / kTmaStages) & 1)) {}
                    const unsigned long long npk = meta_npk[sd], off = meta_off[sd];
                    if (npk == 0) break;                    // end marker reached: everything stored
                    const void* res = data + (size_t)sd * kTmaStageBytes;
                    for (int p = 0; p < n; ++p) bulk_store(P.bufs[p] + off * 16, res, (uint32_t)(npk * 16));
                    bulk_commit();
                }
                if (t >= (unsigned)kTmaStages) bulk_wait_read<1>();   // tile t-S's stores have read stage st
                // next tile into stage st (or the end marker)
                while (!done && pos >= fend) {
                    const unsigned long long k = atomicAdd(g.work, 1ull) - g.wbase;
                    if (k >= g.nchunks) { done = true; break; }
                    const unsigned long long a = g.s0 + (k < g.nbig ? k * g.big : g.bigend + (k - g.nbig) * g.small);
                    unsigned long long b = a + (k < g.nbig ? g.big : g.small);
                    if (b > g.s1) b = g.s1;
                    pos = a;
                    fend = b < g.nfull ? b : (a > g.nfull ? a : g.nfull);
                    if (b > fend) { tail_lo = fend; tail_hi = b; }
                }
                if (done) {
                    meta_npk[st] = 0;
                    mbar_arrive(&full[st]);                 // end marker
                    continue;
                }
                const unsigned long long npk = (fend - pos) < tile_pk ? (fend - pos) : tile_pk;
                meta_off[st] = pos;
                meta_npk[st] = npk;
                mbar_arrive_expect_tx(&full[st], (uint32_t)(n * npk * 16));
                for (int p = 0; p < n; ++p)
                    bulk_load(data + (size_t)st * kTmaStageBytes + p * tile_b, P.bufs[p] + pos * 16,
                              (uint32_t)(npk * 16), &full[st]);
                pos += npk;
            }
            bulk_wait_all();             // every result tile written
            fence_proxy_async_global();  // async-proxy writes ordered before the generic exit flag
            s_tail_lo = tail_lo;
            s_tail_hi = tail_hi;
        }
    } else {
        // ---------------------------------------------------------- consumers
        const unsigned ctid = (unsigned)(tid - 32), cthreads = blockDim.x - 32;
        for (unsigned t = 0;; ++t) {
            const int st = (int)(t % kTmaStages);
            while (!mbar_try_wait(&full[st], (t / kTmaStages) & 1)) {}
            const unsigned long long npk = meta_npk[st];
            if (npk != 0) {
                uint4* tile0 = reinterpret_cast<uint4*>(data + (size_t)st * kTmaStageBytes);
                for (unsigned j = ctid; j < npk; j += cthreads) {
                    Acc<DT> acc;
                    acc_init<DT>(acc, tile0[j]);
                    for (int p = 1; p < n; ++p)
                        acc_add<DT, OP>(acc, reinterpret_cast<const uint4*>(data + (size_t)st * kTmaStageBytes + p * tile_b)[j]);
                    tile0[j] = acc_fin<DT>(acc);
                }
                fence_proxy_async_smem();   // my smem writes -> visible to the bulk store
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            if (npk == 0) break;
        }
    }
    __syncthreads();
    // slow-path remainder (the partial last pack) of a chunk this CTA grabbed
    for (unsigned long long i = s_tail_lo + tid; i < s_tail_hi; i += blockDim.x) {
        Acc<DT> acc;
        acc_init<DT>(acc, load_pack<ES>(P, P.bufs[0], i));
        for (int p = 1; p < n; ++p) acc_add<DT, OP>(acc, load_pack<ES>(P, P.bufs[p], i));
        const uint4 out = acc_fin<DT>(acc);
        for (int p = 0; p < n; ++p) store_pack<ES>(P, P.bufs[p], i, out);
    }
}

// owner j's shard of the zero-copy two-shot as a chunk queue: big chunks first,
// then small ones for the last nch * big packs (balanced tail)
template <int ES>
__device__ __forceinline__ TwoShotGeo twoshot_geo(const Params& P, int j, uint64_t e, unsigned long long big,
                                                  unsigned long long small) {
    TwoShotGeo g;
    g.big = big;
    g.small = small;
    split_range(0, npacks<ES>(P), P.nranks, j, g.s0, g.s1);
    const unsigned long long L = g.s1 - g.s0;
    const unsigned long long tail = L < (unsigned long long)P.nch * big ? L : (unsigned long long)P.nch * big;
    g.nbig = (L - tail) / big;
    g.bigend = g.nbig * big;
    g.nchunks = g.nbig + (L - g.bigend + small - 1) / small;
    g.nfull = P.vec ? (P.count / (16 / ES)) : 0;   // packs safe for the fast path
    g.work = reinterpret_cast<unsigned long long*>(&chan_state(P, j, 0)->work);
    g.wbase = (unsigned long long)e << 32;
    return g;
}

template <int DT, int OP>
__device__ void twoshot_simple(const Params& P, const Who& w) {
    constexpr int ES = DType<DT>::ES;
    const int n = w.n, tid = w.tid;
    ChanState* st = chan_state(P, w.r, w.c);
    const uint64_t e = st->epoch + 1;
    trace_point(P, 0);
    if (!handshake_entry(P, w, e)) return;
    trace_point(P, 1);

    // Owner r's shard [s0, s1) is processed by its nch CTAs with DYNAMIC chunk
    // scheduling: CTAs grab chunk indices from a per-owner counter in the
    // owner's scratch (ChanState[0].work = (epoch << 32) | next), so a slower
    // SM takes fewer chunks (static slices left a ~15 % loop-time spread,
    // measured with polar_comm_set_trace).  Big chunks first, then small ones
    // for the last nch*kTsBig packs so the tail is balanced too.
    const bool tma = P.tma && P.vec;
    const TwoShotGeo g = twoshot_geo<ES>(P, w.r, e, tma ? kTsBigTma : kTsBig, kTsSmall);
    if (tma) {
        twoshot_tma<DT, OP>(P, w, g);
    } else switch (n) {
        case 2: twoshot_loop<DT, OP, 2>(P, w, g); break;
        case 3: twoshot_loop<DT, OP, 3>(P, w, g); break;
        case 4: twoshot_loop<DT, OP, 4>(P, w, g); break;
        default: twoshot_loop<DT, OP, 0>(P, w, g); break;
    }
    __syncthreads();
    trace_point(P, 2);
    if (!handshake_exit(P, w, e)) return;
    trace_point(P, 3);
    epoch_publish(P, w, e);
}

// ====================================================================== wires
// How packs travel through staging slots and FIFOs, per protocol.  A slot is
// addressed by WIRE INDEX k: Simple = one 16-B pack, LL = one pack as two 16-B LL
// lines, LL128 = one warp unit of kLL128Packs packs as a 512-B line group.
// put/get of LL128 are warp-collective (every lane calls them; see for_batch).
//   Simple: payload only; ordering comes from a separate fence + flag.
//   LL    : flag-in-data, flag = (u32) sequence number.
//   LL128 : flag per 128-B line, flag = u64 sequence number.
//
// Latency hiding: every loop moves a BATCH of wire indices per thread
// (Simple / LL) or per warp (LL128) per iteration, and get_batch issues all of
// the batch's loads before it looks at any of them, so several 16-B loads per
// thread are in flight instead of one (Little's law over peer latency).

// Simple moves 4 packs per thread per iteration; LL / LL128 2 (their polls hold
// twice the registers per pack; 4 spilled at the 128-register cap of 512-thread
// CTAs).  bf16 (f32 partials on the wire) halves the batch in ring / tree.
#ifndef POLAR_BATCH_SIMPLE
#define POLAR_BATCH_SIMPLE 4
#endif
#ifndef POLAR_BATCH_LL
#define POLAR_BATCH_LL 2
#endif
#ifndef POLAR_UR_LL128
#define POLAR_UR_LL128 1    // LL128 units per warp in the one-/two-shot reduce (fold_peers)
#endif
template <int PROTO> __host__ __device__ constexpr int batch_for() {
    return PROTO == POLAR_PROTO_SIMPLE ? POLAR_BATCH_SIMPLE : POLAR_BATCH_LL;
}

// One iteration's packs.  Simple / LL: pack i[u] = i0 + u * blockDim, wire index
// j[u] = i[u] - lo.  LL128: unit j[u] = u0 + u * nwarps (warp-uniform), pack
// i[u] = lo + 30 j[u] + lane.  in[u]: the wire index is used (warp-uniform for
// LL128); act[u]: this thread holds a pack of the message.
template <int U> struct Batch {
    unsigned long long i[U], j[U];
    bool in[U], act[U];
};

template <int PROTO> struct Wire;

// Each wire splits a get into issue() (the loads, no waiting), ready() (did this
// thread's copy arrive), decode() and poll() (wait and load again).  Callers issue
// a whole batch — or the same pack from every peer — check readiness once, and
// only if something had not arrived yet fall back to polling each wire index from
// scratch (so no raw value stays live across the out-of-line spin loops).

template <> struct Wire<POLAR_PROTO_SIMPLE> {
    static constexpr unsigned long long kPacks = 1;   // packs per wire index (per thread)
    struct Raw { uint4 a; };
    static __device__ __forceinline__ unsigned long long units(unsigned long long slot_bytes) { return slot_bytes / 16; }
    static __device__ __forceinline__ void put(const Params&, uint4* slot, unsigned long long k, uint4 v, uint64_t) {
        st_plain(slot + k, v);
    }
    static __device__ __forceinline__ void issue(const uint4* slot, unsigned long long k, Raw& r) { r.a = ld_cg(slot + k); }
    static __device__ __forceinline__ bool ready(const Raw&, uint64_t) { return true; }
    static __device__ __forceinline__ uint4 decode(const Raw& r) { return r.a; }
    static __device__ __forceinline__ bool poll(const Params&, const uint4* slot, unsigned long long k, uint64_t, uint4& v) {
        v = ld_cg(slot + k);
        return true;
    }
};
template <> struct Wire<POLAR_PROTO_LL> {
    static constexpr unsigned long long kPacks = 1;
    struct Raw { uint4 a, b; };
    static __device__ __forceinline__ unsigned long long units(unsigned long long slot_bytes) { return slot_bytes / 32; }
    static __device__ __forceinline__ void put(const Params& P, uint4* slot, unsigned long long k, uint4 v, uint64_t f) {
        jitter(P), st_ll(slot + 2 * k, v.x, v.y, (uint32_t)f);
        jitter(P), st_ll(slot + 2 * k + 1, v.z, v.w, (uint32_t)f);
    }
    static __device__ __forceinline__ void issue(const uint4* slot, unsigned long long k, Raw& r) {
        r.a = ld_ll(slot + 2 * k);
        r.b = ld_ll(slot + 2 * k + 1);
    }
    static __device__ __forceinline__ bool ready(const Raw& r, uint64_t f) {
        const uint32_t fl = (uint32_t)f;
        return r.a.y == fl && r.a.w == fl && r.b.y == fl && r.b.w == fl;
    }
    static __device__ __forceinline__ uint4 decode(const Raw& r) { return make_uint4(r.a.x, r.a.z, r.b.x, r.b.z); }
    static __device__ __forceinline__ bool poll(const Params& P, const uint4* slot, unsigned long long k, uint64_t f,
                                                uint4& v) {
        uint4 l0, l1;
        if (!poll_ll(P, slot + 2 * k, (uint32_t)f, l0) || !poll_ll(P, slot + 2 * k + 1, (uint32_t)f, l1)) return false;
        v = make_uint4(l0.x, l0.z, l1.x, l1.z);
        return true;
    }
};
template <> struct Wire<POLAR_PROTO_LL128> {
    static constexpr unsigned long long kPacks = kLL128Packs;
    struct Raw { uint4 a; };
    static __device__ __forceinline__ unsigned long long units(unsigned long long slot_bytes) {
        return slot_bytes / kLL128UnitBytes;
    }
    static __device__ __forceinline__ void put(const Params& P, uint4* slot, unsigned long long k, uint4 v, uint64_t f) {
        jitter_warp(P);
        __syncwarp();
        st_ll128(slot + (kLL128UnitBytes / 16) * k, v, f);
    }
    // warp-collective: every lane issues its 16 B of the line group; ready() is
    // per lane (the caller votes), decode() shuffles
    static __device__ __forceinline__ void issue(const uint4* slot, unsigned long long k, Raw& r) {
        r.a = ld_ll(slot + (kLL128UnitBytes / 16) * k + (threadIdx.x & 31));
    }
    static __device__ __forceinline__ bool ready(const Raw& r, uint64_t f) { return ll128_lane_ready(r.a, f); }
    static __device__ __forceinline__ uint4 decode(const Raw& r) { return ll128_unpack(r.a); }
    static __device__ __forceinline__ bool poll(const Params& P, const uint4* slot, unsigned long long k, uint64_t f,
                                                uint4& v) {
        return ld_ll128(P, slot + (kLL128UnitBytes / 16) * k, f, v);
    }
};

// all-arrived vote: per thread, or per warp for LL128 (whose get is warp-collective)
template <int PROTO> __device__ __forceinline__ bool all_ready(bool mine) {
    if constexpr (PROTO == POLAR_PROTO_LL128) return __all_sync(0xffffffffu, mine);
    return mine;
}

// a batch's NW wire words per pack from one slot
template <int PROTO, int U, int NW>
__device__ __forceinline__ bool get_batch(const Params& P, const uint4* slot, const Batch<U>& b, uint64_t f,
                                          uint4 (&v)[U][NW]) {
    using W = Wire<PROTO>;
    if (PROTO == POLAR_PROTO_LL128) __syncwarp();
    {
        typename W::Raw raw[U][NW];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int q = 0; q < NW; ++q)
                if (b.in[u]) W::issue(slot, b.j[u] * NW + q, raw[u][q]);
        bool rd = true;
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int q = 0; q < NW; ++q)
                if (b.in[u]) rd = rd && W::ready(raw[u][q], f);
        if (all_ready<PROTO>(rd)) {
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int q = 0; q < NW; ++q)
                    if (b.in[u]) v[u][q] = W::decode(raw[u][q]);
            return true;
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
        for (int q = 0; q < NW; ++q)
            if (b.in[u] && !W::poll(P, slot, b.j[u] * NW + q, f, v[u][q])) return false;
    return true;
}

// a batch's NW wire words per pack from nk <= K slots (each with its own flag):
// every slot's loads first, one readiness vote, then decode (tree: both children)
template <int PROTO, int K, int U, int NW>
__device__ __forceinline__ bool get_batch_multi(const Params& P, const uint4* const (&slot)[K], int nk,
                                                const Batch<U>& b, const uint64_t (&f)[K], uint4 (&v)[K][U][NW]) {
    using W = Wire<PROTO>;
    if (PROTO == POLAR_PROTO_LL128) __syncwarp();
    {
        typename W::Raw raw[K][U][NW];
#pragma unroll
        for (int k = 0; k < K; ++k)
            if (k < nk)
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int q = 0; q < NW; ++q)
                        if (b.in[u]) W::issue(slot[k], b.j[u] * NW + q, raw[k][u][q]);
        bool rd = true;
#pragma unroll
        for (int k = 0; k < K; ++k)
            if (k < nk)
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int q = 0; q < NW; ++q)
                        if (b.in[u]) rd = rd && W::ready(raw[k][u][q], f[k]);
        if (all_ready<PROTO>(rd)) {
#pragma unroll
            for (int k = 0; k < K; ++k)
                if (k < nk)
#pragma unroll
                    for (int u = 0; u < U; ++u)
#pragma unroll
                        for (int q = 0; q < NW; ++q)
                            if (b.in[u]) v[k][u][q] = W::decode(raw[k][u][q]);
            return true;
        }
    }
#pragma unroll
    for (int k = 0; k < K; ++k)
        if (k < nk)
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int q = 0; q < NW; ++q)
                    if (b.in[u] && !W::poll(P, slot[k], b.j[u] * NW + q, f[k], v[k][u][q])) return false;
    return true;
}

// Fold the same batch from every rank in rank order: fold(p, u, x) is called for
// p = 0..n-1 (x = own[u] for p == self, else rank p's copy from slot(p)).  All
// loads of all peers are issued first and checked with one vote — one wait for
// n-1 senders instead of n-1 waits; if something has not arrived yet, peers are
// polled one by one in rank order and folded as they arrive (so only the
// accumulators stay live across the out-of-line spin loops).
template <int PROTO, int U, class SlotFn, class Fold>
__device__ __forceinline__ bool fold_peers(const Params& P, SlotFn&& slot, int self, int n, const Batch<U>& b,
                                           uint64_t f, const uint4 (&own)[U], Fold&& fold) {
    using W = Wire<PROTO>;
    if (PROTO == POLAR_PROTO_LL128) __syncwarp();
    {
        typename W::Raw raw[kMaxRanks][U];
#pragma unroll
        for (int p = 0; p < kMaxRanks; ++p)
            if (p < n && p != self)
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (b.in[u]) W::issue(slot(p), b.j[u], raw[p][u]);
        bool rd = true;
#pragma unroll
        for (int p = 0; p < kMaxRanks; ++p)
            if (p < n && p != self)
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (b.in[u]) rd = rd && W::ready(raw[p][u], f);
        if (all_ready<PROTO>(rd)) {
#pragma unroll
            for (int p = 0; p < kMaxRanks; ++p)
                if (p < n)
#pragma unroll
                    for (int u = 0; u < U; ++u) fold(p, u, p == self ? own[u] : W::decode(raw[p][u]));
            return true;
        }
    }
#pragma unroll 1
    for (int p = 0; p < n; ++p)
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint4 x = own[u];
            if (p != self && b.in[u] && !W::poll(P, slot(p), b.j[u], f, x)) return false;
            fold(p, u, x);
        }
    return true;
}

// Run body(batch) over packs [lo, hi) in batches of U (see Batch).  The body
// returns false to stop (timeout); so does for_batch.  For LL128 the whole warp
// runs every iteration (warp-collective wires).
template <int PROTO, int U, class Body>
__device__ __forceinline__ bool for_batch(unsigned long long lo, unsigned long long hi, Body&& body) {
    Batch<U> b;
    if constexpr (PROTO == POLAR_PROTO_LL128) {
        const unsigned lane = threadIdx.x & 31;
        const unsigned long long nw = blockDim.x >> 5;
        for (unsigned long long u0 = threadIdx.x >> 5; lo + u0 * kLL128Packs < hi; u0 += U * nw) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                b.j[u] = u0 + u * nw;
                b.in[u] = lo + b.j[u] * kLL128Packs < hi;
                b.i[u] = lo + b.j[u] * kLL128Packs + lane;
                b.act[u] = b.in[u] && lane < (unsigned)kLL128Packs && b.i[u] < hi;
            }
            if (!body(b)) return false;
        }
    } else {
        const unsigned long long B = blockDim.x;
        for (unsigned long long i0 = lo + threadIdx.x; i0 < hi; i0 += U * B) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                b.i[u] = i0 + u * B;
                b.j[u] = b.i[u] - lo;
                b.in[u] = b.act[u] = b.i[u] < hi;
            }
            if (!body(b)) return false;
        }
    }
    return true;
}

// staging geometry in whole wire units: packs per wire index for PROTO
template <int PROTO>
__device__ __forceinline__ Geo make_geo_for(unsigned long long NP, unsigned long long slot_bytes, int nch, int parts) {
    using W = Wire<PROTO>;
    constexpr unsigned long long unit = PROTO == POLAR_PROTO_LL128 ? (unsigned long long)kLL128Packs : kUnit;
    return make_geo<unit>(NP, W::units(slot_bytes) * W::kPacks, nch, parts);
}

__device__ __forceinline__ uint4 zero4() { return make_uint4(0, 0, 0, 0); }

// own packs of a batch (issued together; zeros where the thread holds no pack)
template <int ES, int U>
__device__ __forceinline__ void load_batch(const Params& P, const char* base, const Batch<U>& b, uint4 (&v)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = b.act[u] ? load_pack<ES>(P, base, b.i[u]) : zero4();
}

// Two-shot LL / LL128: push-based.  RS: rank r writes its part of owner j's
// shard into j's RS staging slot r; owner polls, reduces in rank order, writes
// its own buffer and pushes the result into every rank's AG slot; every rank
// polls the AG slots.  Two NVLink hops, no separate flags.

template <int PROTO>
__device__ __forceinline__ uint4* ts_stage(const Params& P, int owner, int ag, int par, int slot) {
    const unsigned long long base = PROTO == POLAR_PROTO_LL128 ? P.ts128_off : P.tsll_off;
    return reinterpret_cast<uint4*>(P.scratch[owner] + base + (size_t)ag * 2 * kMaxRanks * 2 * P.tsll_chunk +
                                    ((size_t)(par * kMaxRanks + slot)) * 2 * P.tsll_chunk);
}

// shift a batch's wire indices by a staging region offset (in wire units)
template <int U> __device__ __forceinline__ Batch<U> shifted(const Batch<U>& b, unsigned long long ob) {
    Batch<U> s = b;
#pragma unroll
    for (int u = 0; u < U; ++u) s.j[u] += ob;
    return s;
}

template <int DT, int OP, int PROTO>
__device__ void twoshot_ll(const Params& P, const Who& w) {
    constexpr int ES = DType<DT>::ES;
    constexpr int U = batch_for<PROTO>();
    constexpr int UR = PROTO == POLAR_PROTO_LL ? 1 : POLAR_UR_LL128;   // fold_peers holds n-1 raw copies per pack
    using W = Wire<PROTO>;
    const int n = w.n;
    ChanState* st = chan_state(P, w.r, w.c);
    const uint64_t e0 = st->epoch;
    const unsigned long long NP = npacks<ES>(P);
    const Geo g = make_geo_for<PROTO>(NP, 2 * P.tsll_chunk, P.nch, n);
    char* mine = P.bufs[w.r];
    for (unsigned long long k = 0; k < g.nchunks; ++k) {
        const uint64_t e = e0 + k + 1;
        const int par = (int)(e & 1);
        unsigned long long lo, hi, off;
        bool ok = true;
        // RS push: my contribution to every other owner's part
        for (int j = 0; j < n; ++j) {
            if (j == w.r) continue;
            geo_slice(g, NP, k, j, w.c, lo, hi, off);
            uint4* dst = ts_stage<PROTO>(P, j, 0, par, w.r);
            const unsigned long long ob = off / W::kPacks;
            for_batch<PROTO, U>(lo, hi, [&](const Batch<U>& b) {
                uint4 v[U];
                load_batch<ES>(P, mine, b, v);
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (b.in[u]) W::put(P, dst, ob + b.j[u], v[u], e);
                return true;
            });
        }
        // reduce my part in rank order, keep it and push it to every rank; every
        // sender's staging is polled at once (fold_peers); own part only, so this
        // loop may use its own batch (UR) without a barrier
        geo_slice(g, NP, k, w.r, w.c, lo, hi, off);
        const unsigned long long ob = off / W::kPacks;
        ok = for_batch<PROTO, UR>(lo, hi, [&](const Batch<UR>& b) {
            const Batch<UR> sb = shifted(b, ob);
            uint4 own[UR];
            load_batch<ES>(P, mine, b, own);
            Acc<DT> acc[UR];
            if (!fold_peers<PROTO, UR>(
                    P, [&](int p) -> const uint4* { return ts_stage<PROTO>(P, w.r, 0, par, p); }, w.r, n, sb, e, own,
                    [&](int p, int u, const uint4& x) {
                        if (p == 0) acc_init<DT>(acc[u], x);
                        else acc_add<DT, OP>(acc[u], x);
                    }))
                return false;
#pragma unroll
            for (int u = 0; u < UR; ++u) {
                if (!b.in[u]) continue;
                const uint4 out = acc_fin<DT>(acc[u]);
                if (b.act[u]) store_pack<ES>(P, mine, b.i[u], out);
                for (int p = 0; p < n; ++p)
                    if (p != w.r) W::put(P, ts_stage<PROTO>(P, p, 1, par, w.r), sb.j[u], out, e);
            }
            return true;
        });
        // AG receive: results of every other owner
        for (int j = 0; j < n && ok; ++j) {
            if (j == w.r) continue;
            geo_slice(g, NP, k, j, w.c, lo, hi, off);
            const uint4* src = ts_stage<PROTO>(P, w.r, 1, par, j);
            const unsigned long long obj = off / W::kPacks;
            ok = for_batch<PROTO, U>(lo, hi, [&](const Batch<U>& b) {
                uint4 v[U][1];
                if (!get_batch<PROTO, U, 1>(P, src, shifted(b, obj), e, v)) return false;
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (b.act[u]) store_pack<ES>(P, mine, b.i[u], v[u][0]);
                return true;
            });
        }
        if (!__syncthreads_and(ok)) return;   // parity reuse safety
    }
    epoch_publish(P, w, e0 + g.nchunks);
}

// ===================================================================== one-shot
// Every rank pushes its slice to slot r of every peer's staging, then reduces
// slots 0..n-1 in rank order into its own buffer.  One NVLink step;
// egress (n-1)*S.  Chunked through 2 parities when S exceeds a staging slot.

__device__ __forceinline__ uint4* os_slot(const Params& P, int owner, int par, int slot) {
    return reinterpret_cast<uint4*>(P.scratch[owner] + P.os_off + ((size_t)(par * kMaxRanks + slot)) * P.os_chunk);
}
template <int PROTO>
__device__ __forceinline__ uint4* osll_slot(const Params& P, int owner, int par, int slot) {
    const unsigned long long base = PROTO == POLAR_PROTO_LL128 ? P.os128_off : P.osll_off;
    return reinterpret_cast<uint4*>(P.scratch[owner] + base + ((size_t)(par * kMaxRanks + slot)) * 2 * P.osll_chunk);
}

template <int DT, int OP>
__device__ void oneshot_simple(const Params& P, const Who& w) {
    constexpr int ES = DType<DT>::ES;
    constexpr int U = batch_for<POLAR_PROTO_SIMPLE>();
    const int n = w.n, tid = w.tid;
    ChanState* st = chan_state(P, w.r, w.c);
    const uint64_t e0 = st->epoch;
    const unsigned long long NP = npacks<ES>(P);
    const Geo g = make_geo<kUnit>(NP, P.os_chunk / 16, P.nch, 1);
    char* mine = P.bufs[w.r];
    for (unsigned long long k = 0; k < g.nchunks; ++k) {
        const uint64_t e = e0 + k + 1;
        const int par = (int)(e & 1);
        unsigned long long lo, hi, off;
        geo_slice(g, NP, k, 0, w.c, lo, hi, off);
        for_batch<POLAR_PROTO_SIMPLE, U>(lo, hi, [&](const Batch<U>& b) {
            uint4 v[U];
            load_batch<ES>(P, mine, b, v);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (b.in[u])
#pragma unroll
                    for (int p = 0; p < kMaxRanks; ++p)
                        if (p < n && p != w.r) st_plain(os_slot(P, p, par, w.r) + off + b.j[u], v[u]);
            return true;
        });
        __syncthreads();
        if (tid < n && tid != w.r) {
            fence_acq_rel(P.sys);
            jitter(P), st_relaxed(flag_ptr(P, tid, F_OS, w.c, w.r), e, P.sys);
        }
        bool ok = true;
        if (tid < n && tid != w.r) ok = wait_geq(P, flag_ptr(P, w.r, F_OS, w.c, tid), e);
        if (!__syncthreads_and(ok)) return;
        for (unsigned long long i = lo + tid; i < hi; i += blockDim.x) {
            uint4 v[kMaxRanks];
#pragma unroll
            for (int p = 0; p < kMaxRanks; ++p)
                if (p < n) v[p] = (p == w.r) ? load_pack<ES>(P, mine, i) : ld_cg(os_slot(P, w.r, par, p) + off + (i - lo));
            Acc<DT> acc;
            acc_init<DT>(acc, v[0]);
#pragma unroll
            for (int p = 1; p < kMaxRanks; ++p)
                if (p < n) acc_add<DT, OP>(acc, v[p]);
            store_pack<ES>(P, mine, i, acc_fin<DT>(acc));
        }
        if (POLAR_DISCARD) {
            // staging consumed; the peers refill this parity only after our next
            // chunk's (or call's) flag, which the next barrier + fence orders after this
            __syncthreads();
            for (int p = 0; p < n; ++p)
                if (p != w.r) discard_l2(os_slot(P, w.r, par, p) + off, (hi - lo) * 16ull);
        }
    }
    epoch_publish(P, w, e0 + g.nchunks);
}

// one-shot LL / LL128: no separate flags; the data carries them
template <int DT, int OP, int PROTO>
__device__ void oneshot_ll(const Params& P, const Who& w) {
    constexpr int ES = DType<DT>::ES;
    constexpr int U = batch_for<PROTO>();
    constexpr int UR = PROTO == POLAR_PROTO_LL ? 1 : POLAR_UR_LL128;   // fold_peers holds n-1 raw copies per pack
    using W = Wire<PROTO>;
    const int n = w.n;
    ChanState* st = chan_state(P, w.r, w.c);
    const uint64_t e0 = st->epoch;
    const unsigned long long NP = npacks<ES>(P);
    const Geo g = make_geo_for<PROTO>(NP, 2 * P.osll_chunk, P.nch, 1);
    char* mine = P.bufs[w.r];
    bool ok = true;
    for (unsigned long long k = 0; k < g.nchunks; ++k) {
        const uint64_t e = e0 + k + 1;
        const int par = (int)(e & 1);
        unsigned long long lo, hi, off;
        geo_slice(g, NP, k, 0, w.c, lo, hi, off);
        const unsigned long long ob = off / W::kPacks;
        for_batch<PROTO, U>(lo, hi, [&](const Batch<U>& b) {
            uint4 v[U];
            load_batch<ES>(P, mine, b, v);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (b.in[u])
                    for (int p = 0; p < n; ++p)
                        if (p != w.r) W::put(P, osll_slot<PROTO>(P, p, par, w.r), ob + b.j[u], v[u], e);
            return true;
        });
        __syncthreads();   // every push has read `mine` before the reduce below (another batch) writes it
        ok = for_batch<PROTO, UR>(lo, hi, [&](const Batch<UR>& b) {
            const Batch<UR> sb = shifted(b, ob);
            uint4 own[UR];
            load_batch<ES>(P, mine, b, own);
            Acc<DT> acc[UR];
            if (!fold_peers<PROTO, UR>(
                    P, [&](int p) -> const uint4* { return osll_slot<PROTO>(P, w.r, par, p); }, w.r, n, sb, e, own,
                    [&](int p, int u, const uint4& x) {
                        if (p == 0) acc_init<DT>(acc[u], x);
                        else acc_add<DT, OP>(acc[u], x);
                    }))
                return false;
#pragma unroll
            for (int u = 0; u < UR; ++u)
                if (b.act[u]) store_pack<ES>(P, mine, b.i[u], acc_fin<DT>(acc[u]));
            return true;
        });
        if (!__syncthreads_and(ok)) return;   // parity reuse safety
    }
    epoch_publish(P, w, e0 + g.nchunks);
}

// ====================================================================== FIFOs
// A connection is a kSteps-slot FIFO in the RECEIVER's scratch.  The sender
// counts slots sent, the receiver slots consumed; both counters persist in the
// owners' ChanState across calls, so FIFOs never need resetting.
//   Simple: payload, fence, tail flag (= sent) in the receiver's scratch.
//   LL    : payload as LL lines whose flag is (u32)(slot sequence + 1).
//   LL128 : payload as LL128 line groups whose flag is slot sequence + 1.
//   All   : the receiver returns a head credit (= consumed) to the sender.
// The three protocols share the counters and flags but not the FIFO memory.

template <int PROTO> __device__ __forceinline__ unsigned long long ring_slot_bytes(const Params& P) {
    return PROTO == POLAR_PROTO_LL ? P.ringll_slot : PROTO == POLAR_PROTO_LL128 ? P.ring128_slot : P.ring_slot;
}
template <int PROTO> __device__ __forceinline__ unsigned long long tree_slot_bytes(const Params& P) {
    return PROTO == POLAR_PROTO_LL ? P.treell_slot : PROTO == POLAR_PROTO_LL128 ? P.tree128_slot : P.tree_slot;
}

// ======================================================================= ring
// nch rings in rank order.  Per channel, loop chunks of n sub-chunks; step s of
// reduce-scatter sends sub-chunk (r - s) mod n to r+1; after n-1 steps rank r
// holds the full reduction of sub-chunk r+1; n-1 all-gather steps forward it.

template <int PROTO>
__device__ __forceinline__ uint4* ring_slot(const Params& P, int owner, int c, unsigned long long seq) {
    const unsigned long long off =
        PROTO == POLAR_PROTO_LL ? P.ringll_off : PROTO == POLAR_PROTO_LL128 ? P.ring128_off : P.ring_off;
    return reinterpret_cast<uint4*>(P.scratch[owner] + off + ((size_t)c * kSteps + (seq % kSteps)) * ring_slot_bytes<PROTO>(P));
}

template <int DT, int OP, int PROTO>
__device__ void ring(const Params& P, const Who& w) {
    constexpr int ES = DType<DT>::ES;
    constexpr int AW = AccWords<DT>::N;
    constexpr int U = batch_for<PROTO>() / AW > 0 ? batch_for<PROTO>() / AW : 1;
    using W = Wire<PROTO>;
    const int n = w.n, tid = w.tid, r = w.r, c = w.c;
    const int next = (r + 1) % n, prev = (r + n - 1) % n;
    ChanState* st = chan_state(P, r, c);
    unsigned long long sent = st->ring_sent, recvd = st->ring_recv;
    // element packs per slot: AW wire indices per pack (f32 partials of bf16)
    const unsigned long long SP = W::units(ring_slot_bytes<PROTO>(P)) / AW * W::kPacks;
    const unsigned long long NP = npacks<ES>(P);
    unsigned long long ca, cb;
    split_range(0, NP, P.nch, c, ca, cb);
    char* mine = P.bufs[r];
    uint64_t* head_in = flag_ptr(P, r, F_RING_HEAD, c, 0);     // credits from next
    uint64_t* tail_in = flag_ptr(P, r, F_RING_TAIL, c, 0);     // fills from prev (Simple)
    uint64_t* tail_out = flag_ptr(P, next, F_RING_TAIL, c, 0);
    uint64_t* head_out = flag_ptr(P, prev, F_RING_HEAD, c, 0);
    const unsigned long long LC = SP * (unsigned long long)n;
    for (unsigned long long base = ca; base < cb; base += LC) {
        const unsigned long long L = (cb - base < LC) ? cb - base : LC;
        for (int s = 0; s < 2 * (n - 1) + 1; ++s) {
            const bool do_recv = s > 0;
            const bool do_send = s < 2 * (n - 1);
            // sub-chunk handled at this step
            int k;
            if (s < n) k = ((r - s) % n + n) % n;           // RS steps (s = n-1 finalizes k = r+1)
            else k = ((r - (s - n) ) % n + n) % n;          // AG step t = s-n receives chunk r - t
            if (s == n - 1) k = (r + 1) % n;
            const unsigned long long ks = base + L * (unsigned long long)k / n;
            const unsigned long long ke = base + L * (unsigned long long)(k + 1) / n;
            // ---- waits (thread 0: the fill from prev, thread 1: the credit from next), then barrier
            bool ok = true;
            if (tid == 0 && do_recv && PROTO == POLAR_PROTO_SIMPLE) ok = wait_geq(P, tail_in, recvd + 1);
            if (tid == 1 && do_send && sent >= (unsigned long long)kSteps) ok = wait_geq(P, head_in, sent - kSteps + 1);
            if (!__syncthreads_and(ok)) return;
            const uint4* src = ring_slot<PROTO>(P, r, c, recvd);
            uint4* dst = ring_slot<PROTO>(P, next, c, sent);
            const uint64_t fin = recvd + 1, fout = sent + 1;
            ok = for_batch<PROTO, U>(ks, ke, [&](const Batch<U>& b) {
                uint4 own[U];
                if (s < n) load_batch<ES>(P, mine, b, own);
                if (s == 0) {
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        if (!b.in[u]) continue;
                        Acc<DT> acc;
                        acc_init<DT>(acc, own[u]);
#pragma unroll
                        for (int q = 0; q < AW; ++q) W::put(P, dst, b.j[u] * AW + q, acc.w[q], fout);
                    }
                } else if (s < n) {
                    uint4 in[U][AW];
                    if (!get_batch<PROTO, U, AW>(P, src, b, fin, in)) return false;
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        if (!b.in[u]) continue;
                        Acc<DT> acc;
#pragma unroll
                        for (int q = 0; q < AW; ++q) acc.w[q] = in[u][q];
                        if (b.act[u]) acc_add<DT, OP>(acc, own[u]);
                        if (s < n - 1) {
#pragma unroll
                            for (int q = 0; q < AW; ++q) W::put(P, dst, b.j[u] * AW + q, acc.w[q], fout);
                        } else {
                            const uint4 out = acc_fin<DT>(acc);
                            if (b.act[u]) store_pack<ES>(P, mine, b.i[u], out);
                            W::put(P, dst, b.j[u], out, fout);
                        }
                    }
                } else {
                    uint4 v[U][1];
                    if (!get_batch<PROTO, U, 1>(P, src, b, fin, v)) return false;
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        if (!b.in[u]) continue;
                        if (b.act[u]) store_pack<ES>(P, mine, b.i[u], v[u][0]);
                        if (do_send) W::put(P, dst, b.j[u], v[u][0], fout);
                    }
                }
                return true;
            });
            if (!__syncthreads_and(ok)) return;
            if (PROTO == POLAR_PROTO_SIMPLE && POLAR_DISCARD && do_recv) {
                // the slot is consumed: drop its lines before the credit frees it
                discard_l2(src, (ke - ks) * (unsigned long long)(s < n ? AW : 1) * 16ull);
                __syncthreads();
            }
            if (tid == 0) {
                if (PROTO == POLAR_PROTO_SIMPLE && (do_send || (POLAR_DISCARD && do_recv))) fence_acq_rel(P.sys);
                if (do_send && PROTO == POLAR_PROTO_SIMPLE) jitter(P), st_relaxed(tail_out, sent + 1, P.sys);
                if (do_recv) jitter(P), st_relaxed(head_out, recvd + 1, P.sys);
            }
            if (do_send) ++sent;
            if (do_recv) ++recvd;
        }
    }
    if (tid == 0) {
        st->ring_sent = sent;
        st->ring_recv = recvd;
    }
}

// Ring Simple, warp specialised (POLAR_RING_WS).  Measured on the plain ring
// above: every step's synchronisation point (barrier, fence, tail flag, the
// successor's poll) costs ~1.8 us of L2 round trips even when nothing waits, and
// the ring runs in lock-step, so each step pays it on top of its data time
// (DESIGN.md "Ring on virtual ranks").  Here warp 0 is a synchronisation warp
// and warps 1.. move data:
//   * the slot travels in RQ sub-slices (units), each published by its own tail
//     value (sent * RQ + q + 1), so a successor starts a step while its producer
//     is still filling the step's later sub-slices;
//   * the sync warp polls unit g's fill flag (and, at a step's first unit, the
//     credit) and hands the unit to the data warps with bar.arrive READY[g&1];
//     it then waits DONE[(g-1)&1] and publishes unit g-1 (fence, tail; the
//     credit after a step's last unit) — polls and fences run while the data
//     warps already move unit g;
//   * data warps: bar.sync READY[g&1], move the unit, bar.arrive DONE[g&1].
// Two barrier ids per direction suffice: the sync warp arrives READY for unit g
// only after DONE of unit g-2 completed (so every data warp passed READY of
// g-2), and data warps arrive DONE for g+2 only after READY of g+2, which the sync
// warp arrives after it consumed DONE of g.  Only the sync warp spins; on a
// timeout it raises s_abort before its arrive and leaves, and the data warps leave
// at the next READY.
#ifndef POLAR_RING_WS
#define POLAR_RING_WS 1
#endif
#ifndef POLAR_RING_WS_SUB
#define POLAR_RING_WS_SUB 2
#endif
#ifndef POLAR_RING_WS_BATCH
#define POLAR_RING_WS_BATCH POLAR_BATCH_SIMPLE   // packs per data thread per iteration (f32)
#endif
#ifndef POLAR_WS_PREFETCH
#define POLAR_WS_PREFETCH 0
#endif
// The sync warp warms L2 with the data warps' NEXT own-buffer range (ring
// reduce-scatter steps, tree up slots): one cp.async.bulk.prefetch.L2 per 32 KiB,
// no registers, so the data warps' own loads hit L2 instead of HBM.  Only full,
// 16-B aligned packs (P.vec; the partial last pack is never prefetched).
// Off by default: measured no gain (profiles/r01_ws_prefetch_ab.jsonl: ring
// 128 MiB 927 -> 932 us, 1 MiB 39.9 -> 43.3 us; tree 128 MiB 1100 -> 1083 us) —
// the data warps are not waiting on their own-buffer loads.
__device__ __forceinline__ void prefetch_own(const Params& P, const char* base, unsigned long long a,
                                             unsigned long long b, unsigned long long full) {
#if POLAR_WS_PREFETCH
    if (!P.vec) return;
    if (b > full) b = full;
    for (unsigned long long o = a; o < b; o += 2048) {
        const unsigned long long e = (b - o < 2048) ? b - o : 2048;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + o * 16), "r"((unsigned)(e * 16)) : "memory");
    }
#endif
}
// wait_geq with a per-lane cache of the last value acquired from *p (monotone
// flags): skips the load when an earlier acquire already covers v (that acquire
// still orders everything after it)
#ifndef POLAR_WS_CACHED_POLL
#define POLAR_WS_CACHED_POLL 1
#endif
__device__ __forceinline__ bool wait_cached(const Params& P, const uint64_t* p, uint64_t v, uint64_t& seen) {
    if (POLAR_WS_CACHED_POLL && seen >= v) return true;
    seen = ld_acquire(p, P.sys);
    if (seen >= v) return true;
    if (!wait_geq_slow(p, v, P.sys, P.timeout_ns, P.err)) return false;
    seen = v;
    return true;
}
__device__ __forceinline__ void nbar_sync(int id, int cnt) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int cnt) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }

template <int DT, int OP>
__device__ void ring_simple_ws(const Params& P, const Who& w) {
    constexpr int ES = DType<DT>::ES;
    constexpr int AW = AccWords<DT>::N;
    constexpr int U = POLAR_RING_WS_BATCH / AW > 0 ? POLAR_RING_WS_BATCH / AW : 1;
    constexpr int RQ = POLAR_RING_WS_SUB;
    // unit g's fill was published by the predecessor at ITS unit g - RQ, and a
    // rank publishes unit g - 1 only after its waits for unit g: RQ = 1 would make
    // every rank wait for its predecessor's wait around the ring (measured: timeout)
    static_assert(RQ >= 2, "the publication lag needs >= 2 sub-slices per slot");
    constexpr int kReady = 1, kDone = 3;          // named barrier ids (0 is __syncthreads)
    using W = Wire<POLAR_PROTO_SIMPLE>;
    const int n = w.n, tid = w.tid, r = w.r, c = w.c;
    const int next = (r + 1) % n, prev = (r + n - 1) % n;
    const int nthr = blockDim.x;
    ChanState* st = chan_state(P, r, c);
    unsigned long long sent = st->ring_sent, recvd = st->ring_recv;
    const unsigned long long SP = W::units(P.ring_slot) / AW;   // element packs per slot
    const unsigned long long NP = npacks<ES>(P);
    unsigned long long ca, cb;
    split_range(0, NP, P.nch, c, ca, cb);
    char* mine = P.bufs[r];
    const unsigned long long LC = SP * (unsigned long long)n;
    const unsigned long long full_packs = P.count * (unsigned long long)ES / 16;   // whole 16-B packs
    __shared__ int s_abort;
    if (tid == 0) s_abort = 0;
    __syncthreads();

    if (tid < 32) {
        // ---------------------------------------------------------- sync warp
        const int lane = tid;
        uint64_t* head_in = flag_ptr(P, r, F_RING_HEAD, c, 0);    // credits from next
        uint64_t* tail_in = flag_ptr(P, r, F_RING_TAIL, c, 0);    // fills from prev
        uint64_t* tail_out = flag_ptr(P, next, F_RING_TAIL, c, 0);
        uint64_t* head_out = flag_ptr(P, prev, F_RING_HEAD, c, 0);
        unsigned long long g = 0;
        uint64_t seen = 0;                                // lane 0: last fill, lane 1: last credit acquired
        uint64_t pub_tail = 0, pub_head = 0;              // unit g-1's flag values (0: none)
        auto publish = [&]() {
            nbar_sync(kDone + (int)((g - 1) & 1), nthr);  // unit g-1 moved by every data warp
            if (lane == 0) {
                fence_acq_rel(P.sys);
                if (pub_tail) jitter(P), st_relaxed(tail_out, pub_tail, P.sys);
                if (pub_head) jitter(P), st_relaxed(head_out, pub_head, P.sys);
            }
        };
        for (unsigned long long base = ca; base < cb; base += LC) {
            for (int s = 0; s < 2 * (n - 1) + 1; ++s) {
                const bool do_recv = s > 0, do_send = s < 2 * (n - 1);
                for (int q = 0; q < RQ; ++q) {
                    // lane 0: the fill, lane 1: the credit, in parallel; each lane
                    // keeps the last value it acquired (flags are monotone), so a
                    // unit already covered by an earlier load costs no round trip
                    int ok = 1;
                    if (lane == 0 && do_recv) ok = wait_cached(P, tail_in, recvd * RQ + q + 1, seen);
                    if (lane == 1 && q == 0 && do_send && sent >= (unsigned long long)kSteps)
                        ok = wait_cached(P, head_in, sent - kSteps + 1, seen);
                    ok = __all_sync(0xffffffffu, ok);
                    if (!ok && lane == 0) *(volatile int*)&s_abort = 1;
                    __syncwarp();
                    nbar_arrive(kReady + (int)(g & 1), nthr);
                    if (!ok) return;
                    if (g > 0) publish();
                    if (POLAR_WS_PREFETCH && lane == 0 && q == 0) {
                        // own slice of the next reduce-scatter step (or the next lap's step 0)
                        const bool nxt_lap = s == 2 * (n - 1);
                        if (s + 1 < n || nxt_lap) {
                            const unsigned long long b2 = nxt_lap ? base + LC : base;
                            if (b2 < cb) {
                                const unsigned long long L2 = (cb - b2 < LC) ? cb - b2 : LC;
                                const int k2 = nxt_lap ? r : ((r - (s + 1)) % n + n) % n;
                                prefetch_own(P, mine, b2 + L2 * (unsigned long long)k2 / n,
                                             b2 + L2 * (unsigned long long)(k2 + 1) / n, full_packs);
                            }
                        }
                    }
                    pub_tail = do_send ? sent * RQ + q + 1 : 0;
                    pub_head = (do_recv && q == RQ - 1) ? recvd + 1 : 0;
                    ++g;
                }
                if (do_send) ++sent;
                if (do_recv) ++recvd;
            }
        }
        if (g > 0) publish();
        if (lane == 0) {
            st->ring_sent = sent;
            st->ring_recv = recvd;
        }
        return;
    }
    // -------------------------------------------------------------- data warps
    const unsigned long long D = (unsigned long long)(nthr - 32), dt = (unsigned long long)(tid - 32);
    unsigned long long g = 0;
    for (unsigned long long base = ca; base < cb; base += LC) {
        const unsigned long long L = (cb - base < LC) ? cb - base : LC;
        for (int s = 0; s < 2 * (n - 1) + 1; ++s) {
            const bool do_send = s < 2 * (n - 1);
            int k;
            if (s < n) k = ((r - s) % n + n) % n;
            else k = ((r - (s - n)) % n + n) % n;
            if (s == n - 1) k = (r + 1) % n;
            const unsigned long long ks = base + L * (unsigned long long)k / n;
            const unsigned long long ke = base + L * (unsigned long long)(k + 1) / n;
            const uint4* src = ring_slot<POLAR_PROTO_SIMPLE>(P, r, c, recvd);
            uint4* dst = ring_slot<POLAR_PROTO_SIMPLE>(P, next, c, sent);
            for (int q = 0; q < RQ; ++q) {
                const unsigned long long qs = ks + (ke - ks) * (unsigned long long)q / RQ;
                const unsigned long long qe = ks + (ke - ks) * (unsigned long long)(q + 1) / RQ;
                nbar_sync(kReady + (int)(g & 1), nthr);
                if (*(volatile int*)&s_abort) return;
                for (unsigned long long i0 = qs + dt; i0 < qe; i0 += U * D) {
                    Batch<U> b;
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        b.i[u] = i0 + u * D;
                        b.j[u] = b.i[u] - ks;               // wire index in the slot
                        b.in[u] = b.act[u] = b.i[u] < qe;
                    }
                    uint4 own[U];
                    if (s < n) load_batch<ES>(P, mine, b, own);
                    if (s == 0) {
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            if (!b.in[u]) continue;
                            Acc<DT> acc;
                            acc_init<DT>(acc, own[u]);
#pragma unroll
                            for (int x = 0; x < AW; ++x) W::put(P, dst, b.j[u] * AW + x, acc.w[x], 0);
                        }
                    } else if (s < n) {
                        uint4 in[U][AW];
#pragma unroll
                        for (int u = 0; u < U; ++u)
#pragma unroll
                            for (int x = 0; x < AW; ++x)
                                if (b.in[u]) in[u][x] = ld_cg(src + b.j[u] * AW + x);
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            if (!b.in[u]) continue;
                            Acc<DT> acc;
#pragma unroll
                            for (int x = 0; x < AW; ++x) acc.w[x] = in[u][x];
                            acc_add<DT, OP>(acc, own[u]);
                            if (s < n - 1) {
#pragma unroll
                                for (int x = 0; x < AW; ++x) W::put(P, dst, b.j[u] * AW + x, acc.w[x], 0);
                            } else {
                                const uint4 out = acc_fin<DT>(acc);
                                store_pack<ES>(P, mine, b.i[u], out);
                                W::put(P, dst, b.j[u], out, 0);
                            }
                        }
                    } else {
                        uint4 v[U];
#pragma unroll
                        for (int u = 0; u < U; ++u)
                            if (b.in[u]) v[u] = ld_cg(src + b.j[u]);
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            if (!b.in[u]) continue;
                            store_pack<ES>(P, mine, b.i[u], v[u]);
                            if (do_send) W::put(P, dst, b.j[u], v[u], 0);
                        }
                    }
                }
                nbar_arrive(kDone + (int)(g & 1), nthr);
                ++g;
            }
            if (do_send) ++sent;
            if (s > 0) ++recvd;
        }
    }
}


// Ring Simple, TMA-staged (POLAR_RING_TMA).  The warp-specialised
// ring above is limited by loads in flight per data thread (ncu: 40 % long-
// scoreboard stalls, L2 36 % / DRAM 53 % of peak) and the register cap.  Here
// the FIFO and own-buffer traffic moves as cp.async.bulk copies through
// shared-memory stages, so bytes in flight cost no registers:
//   warp 0  sync     : unchanged role (polls fills / credits, hands a unit over
//                      with READY, publishes unit g-1 after DONE(g-1))
//   warp 1  loader   : after READY(g), per tile of unit g: one bulk load of the
//                      predecessor's FIFO words and one of my own packs into a
//                      stage (`full` mbarrier counts the bytes)
//   warp 2  storer   : per tile, once the consumers are done (`cons`): bulk
//                      stores of the result to the successor's FIFO and/or my
//                      buffer; frees a stage once its stores have read it
//                      (`empty`, lagged by one tile); at a unit's end waits for
//                      its writes (wait_group 0 + proxy fence) and arrives DONE(g)
//   warps 3+ consumers: reduce in shared memory (reduce-scatter steps only)
// Tile kinds per step s (AW = accumulator words: 2 for bf16's f32 partials):
//   s = 0        own -> [widen] -> next FIFO (AW words)
//   0 < s < n-1  FIFO (AW) (op) own -> next FIFO (AW)
//   s = n-1      fin(FIFO (AW) (op) own) -> own buffer + next FIFO (1 word)
//   s >= n       FIFO (1) -> own buffer (+ next FIFO unless last)  (no compute)
// Same units, tails, credits and slot layout as ring_simple_ws, so the two
// kernels share FIFOs and counters across calls; used when every pack is a
// full 16-B pack of a 16-B aligned buffer (bulk copies are 16-B granular),
// else ring_simple_ws runs.
#ifndef POLAR_RING_TMA
#define POLAR_RING_TMA 1
#endif
// (stage geometry: device.cuh kRtStages / kRtTile / ring_tma_smem_bytes)

// Walk the ring schedule of one channel exactly as ring_simple_ws does: for each
// unit (sub-slice q of step s of a lap) call unit(g, s, q, ...), and for each
// tile of it tile(t, s, i0, npk, j0, src, dst).  Every role of the kernel walks
// the same sequence, so tile t and unit g mean the same thing to all of them.
template <int DT, class FU, class FT>
__device__ __forceinline__ bool ring_tma_walk(const Params& P, int r, int n, int c, unsigned long long ca,
                                              unsigned long long cb, unsigned long long SP, unsigned long long sent,
                                              unsigned long long recvd, FU&& unit, FT&& tile) {
    constexpr int RQ = POLAR_RING_WS_SUB;
    const int next = (r + 1) % n;
    const unsigned long long LC = SP * (unsigned long long)n;
    unsigned long long g = 0, t = 0;
    for (unsigned long long base = ca; base < cb; base += LC) {
        const unsigned long long L = (cb - base < LC) ? cb - base : LC;
        for (int s = 0; s < 2 * (n - 1) + 1; ++s) {
            int k;
            if (s < n) k = ((r - s) % n + n) % n;
            else k = ((r - (s - n)) % n + n) % n;
            if (s == n - 1) k = (r + 1) % n;
            const unsigned long long ks = base + L * (unsigned long long)k / n;
            const unsigned long long ke = base + L * (unsigned long long)(k + 1) / n;
            const uint4* src = ring_slot<POLAR_PROTO_SIMPLE>(P, r, c, recvd);
            uint4* dst = ring_slot<POLAR_PROTO_SIMPLE>(P, next, c, sent);
            for (int q = 0; q < RQ; ++q) {
                const unsigned long long qs = ks + (ke - ks) * (unsigned long long)q / RQ;
                const unsigned long long qe = ks + (ke - ks) * (unsigned long long)(q + 1) / RQ;
                if (!unit(g, s, q, true)) return false;
                for (unsigned long long i0 = qs; i0 < qe; i0 += kRtTile) {
                    const unsigned npk = (unsigned)((qe - i0) < kRtTile ? (qe - i0) : kRtTile);
                    if (!tile(t, s, i0, npk, i0 - ks, src, dst)) return false;
                    ++t;
                }
                if (!unit(g, s, q, false)) return false;
                ++g;
            }
            if (s < 2 * (n - 1)) ++sent;
            if (s > 0) ++recvd;
        }
    }
    return true;
}

template <int DT, int OP>
__device__ void ring_simple_tma(const Params& P, const Who& w) {
    constexpr int AW = AccWords<DT>::N;
    constexpr int RQ = POLAR_RING_WS_SUB;
    static_assert(RQ >= 2, "the publication lag needs >= 2 sub-slices per slot");
    constexpr int kReady = 1, kDone = 3;
    const int n = w.n, tid = w.tid, r = w.r, c = w.c;
    const int next = (r + 1) % n, prev = (r + n - 1) % n;
    const int warp = tid >> 5, lane = tid & 31;
    ChanState* st = chan_state(P, r, c);
    const unsigned long long sent0 = st->ring_sent, recvd0 = st->ring_recv;
    const unsigned long long SP = Wire<POLAR_PROTO_SIMPLE>::units(P.ring_slot) / AW;   // element packs per slot
    unsigned long long ca, cb;
    split_range(0, npacks<DType<DT>::ES>(P), P.nch, c, ca, cb);
    char* mine = P.bufs[r];
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)kRtStages * kRtStageBytes);
    uint64_t* cons = full + kRtStages;
    uint64_t* empty = cons + kRtStages;
    const int ncons_warps = (int)(blockDim.x >> 5) - 3;
    __shared__ int s_abort;
    if (tid == 0) {
        s_abort = 0;
        for (int x = 0; x < kRtStages; ++x) {
            mbar_init(&full[x], 1);
            mbar_init(&cons[x], (uint32_t)ncons_warps);
            mbar_init(&empty[x], 1);
        }
        mbar_fence_init();
    }
    __syncthreads();
    auto in_smem = [&](unsigned long long t) { return smem + (size_t)(t % kRtStages) * kRtStageBytes; };
    auto own_smem = [&](unsigned long long t) { return smem + (size_t)(t % kRtStages) * kRtStageBytes + kRtInBytes; };
    auto in_words = [&](int s) { return s == 0 ? 0 : (s <= n - 1 ? AW : 1); };

    if (warp == 0) {
        // ------------------------------------------------------------ sync warp
        uint64_t* head_in = flag_ptr(P, r, F_RING_HEAD, c, 0);
        uint64_t* tail_in = flag_ptr(P, r, F_RING_TAIL, c, 0);
        uint64_t* tail_out = flag_ptr(P, next, F_RING_TAIL, c, 0);
        uint64_t* head_out = flag_ptr(P, prev, F_RING_HEAD, c, 0);
        unsigned long long sent = sent0, recvd = recvd0, gpub = 0;
        uint64_t seen = 0, pub_tail = 0, pub_head = 0;
        auto publish = [&]() {
            nbar_sync(kDone + (int)((gpub - 1) & 1), 64);   // unit g-1's writes are complete (storer)
            if (lane == 0) {
                fence_acq_rel(P.sys);
                if (pub_tail) jitter(P), st_relaxed(tail_out, pub_tail, P.sys);
                if (pub_head) jitter(P), st_relaxed(head_out, pub_head, P.sys);
            }
        };
        const bool ok = ring_tma_walk<DT>(P, r, n, c, ca, cb, SP, sent0, recvd0,
            [&](unsigned long long g, int s, int q, bool begin) {
                if (!begin) {
                    if (q == RQ - 1) {
                        if (s < 2 * (n - 1)) ++sent;
                        if (s > 0) ++recvd;
                    }
                    return true;
                }
                const bool do_recv = s > 0, do_send = s < 2 * (n - 1);
                int okw = 1;
                if (lane == 0 && do_recv) okw = wait_cached(P, tail_in, recvd * RQ + q + 1, seen);
                if (lane == 1 && q == 0 && do_send && sent >= (unsigned long long)kSteps)
                    okw = wait_cached(P, head_in, sent - kSteps + 1, seen);
                okw = __all_sync(0xffffffffu, okw);
                if (!okw && lane == 0) *(volatile int*)&s_abort = 1;
                __syncwarp();
                nbar_arrive(kReady + (int)(g & 1), 64);
                if (!okw) return false;
                if (g > 0) publish();
                pub_tail = do_send ? sent * RQ + q + 1 : 0;
                pub_head = (do_recv && q == RQ - 1) ? recvd + 1 : 0;
                gpub = g + 1;
                return true;
            },
            [&](unsigned long long, int, unsigned long long, unsigned, unsigned long long, const uint4*, uint4*) {
                return true;
            });
        if (!ok) return;
        if (gpub > 0) publish();
        if (lane == 0) {
            st->ring_sent = sent;
            st->ring_recv = recvd;
        }
        return;
    }
    if (warp == 1) {
        // -------------------------------------------------------------- loader
        unsigned long long issued = 0;   // tiles issued so far
        const uint64_t pol_first = l2_evict_first();
        const bool ok = ring_tma_walk<DT>(P, r, n, c, ca, cb, SP, sent0, recvd0,
            [&](unsigned long long g, int, int, bool begin) {
                if (!begin) return true;
                nbar_sync(kReady + (int)(g & 1), 64);
                if (*(volatile int*)&s_abort) return false;
                if (lane == 0) fence_proxy_async_global();   // the fills acquired by the sync warp -> bulk reads
                return true;
            },
            [&](unsigned long long t, int s, unsigned long long i0, unsigned npk, unsigned long long j0,
                const uint4* src, uint4*) {
                int ab = 0;
                if (lane == 0) {
                    const int x = (int)(t % kRtStages);
                    if (t >= (unsigned long long)kRtStages)
                        while (!mbar_try_wait(&empty[x], (uint32_t)((t / kRtStages - 1) & 1)))
                            if (*(volatile int*)&s_abort) { ab = 1; break; }
                }
                if (__shfl_sync(0xffffffffu, ab, 0)) return false;
                if (lane == 0) {
                    const int x = (int)(t % kRtStages);
                    const int wi = in_words(s);
                    const bool own = s <= n - 1;
                    const uint32_t bin = npk * 16u * (uint32_t)wi, bown = own ? npk * 16u : 0u;
                    mbar_arrive_expect_tx(&full[x], bin + bown);
                    const char* fsrc = reinterpret_cast<const char*>(src) + j0 * 16ull * wi;
                    if (P.ring_flags & 1) {
                        // both are read once here: evict first
                        if (bin) bulk_load_hint(in_smem(t), fsrc, bin, &full[x], pol_first);
                        if (bown) bulk_load_hint(own_smem(t), mine + i0 * 16ull, bown, &full[x], pol_first);
                    } else {
                        if (bin) bulk_load(in_smem(t), fsrc, bin, &full[x]);
                        if (bown) bulk_load(own_smem(t), mine + i0 * 16ull, bown, &full[x]);
                    }
                }
                issued = t + 1;
                return true;
            });
        if (!ok && lane == 0) {
            // aborted (a peer timed out): every bulk load issued must land before
            // this CTA's shared memory goes away; no newer phase is ever started
            const unsigned long long lo = issued > (unsigned long long)kRtStages ? issued - kRtStages : 0;
            for (unsigned long long t = lo; t < issued; ++t)
                while (!mbar_try_wait(&full[t % kRtStages], (uint32_t)((t / kRtStages) & 1))) {}
        }
        return;
    }
    if (warp == 2) {
        // -------------------------------------------------------------- storer
        long long pending = -1;   // tile whose stage is released once its stores have read it
        const uint64_t pol_first = l2_evict_first(), pol_last = l2_evict_last();
        // DONE(g) once unit g's writes are complete.  (Arriving it lazily, after
        // the next unit's first tile with wait_group 1, was measured slower: the
        // later publication lengthens every hop of the ring's chain — 8 MiB
        // 85 -> 106 us, 128 MiB 1079 -> 1128 us; profiles/r02_ring_tma_ab.jsonl.)
        ring_tma_walk<DT>(P, r, n, c, ca, cb, SP, sent0, recvd0,
            [&](unsigned long long g, int, int, bool begin) {
                if (begin) return true;
                if (lane == 0) {
                    bulk_wait_all();                   // unit g's writes are complete
                    if (pending >= 0) mbar_arrive(&empty[pending % kRtStages]);
                    fence_proxy_async_global();        // async-proxy writes -> the sync warp's fence + flag
                }
                pending = -1;
                __syncwarp();
                nbar_arrive(kDone + (int)(g & 1), 64);
                return true;
            },
            [&](unsigned long long t, int s, unsigned long long i0, unsigned npk, unsigned long long j0,
                const uint4* src, uint4* dst) {
                const int x = (int)(t % kRtStages);
                int ab = 0;
                if (lane == 0) {
                    while (!mbar_try_wait(&cons[x], (uint32_t)((t / kRtStages) & 1)))
                        if (*(volatile int*)&s_abort) break;
                    ab = *(volatile int*)&s_abort;
                }
                ab = __shfl_sync(0xffffffffu, ab, 0);
                if (!ab && (P.ring_flags & 2) && s > 0) {
                    // The tile's FIFO words are in shared memory now (cons implies the
                    // loads landed) and the slot is rewritten by the predecessor only
                    // after our credit: drop its lines from L2 without write-back
                    // (whole 128-B lines inside the tile only: a boundary line may
                    // hold words of a neighbour tile not loaded yet).
                    const int wi = in_words(s);
                    const unsigned long long a = reinterpret_cast<unsigned long long>(src) + j0 * 16ull * wi;
                    const unsigned long long e = a + (unsigned long long)npk * 16ull * wi;
                    for (unsigned long long l = ((a + 127) & ~127ull) + (unsigned long long)lane * 128; l + 128 <= e;
                         l += 32 * 128)
                        asm volatile("discard.global.L2 [%0], 128;" ::"l"(l) : "memory");
                    __syncwarp();
                }
                if (lane == 0) {
                    if (!ab) {
                        const bool first = s == 0, fin = s == n - 1, ag = s >= n;
                        const bool send = s < 2 * (n - 1);
                        // which stage region holds the result, and how many words per pack
                        const void* res;
                        int wo;
                        if (fin) { res = own_smem(t); wo = 1; }
                        else if (ag) { res = in_smem(t); wo = 1; }
                        else if (first && AW == 1) { res = own_smem(t); wo = 1; }
                        else { res = in_smem(t); wo = AW; }
                        char* fdst = reinterpret_cast<char*>(dst) + j0 * 16ull * wo;
                        if (P.ring_flags & 1) {
                            // FIFO words are read soon by the successor: keep them; my result is streaming
                            if (send) bulk_store_hint(fdst, res, npk * 16u * (uint32_t)wo, pol_last);
                            if (fin || ag) bulk_store_hint(mine + i0 * 16ull, res, npk * 16u, pol_first);
                        } else {
                            if (send) bulk_store(fdst, res, npk * 16u * (uint32_t)wo);
                            if (fin || ag) bulk_store(mine + i0 * 16ull, res, npk * 16u);
                        }
                        bulk_commit();
                        bulk_wait_read<1>();               // the previous tile's stores have read its stage
                        if (pending >= 0) mbar_arrive(&empty[pending % kRtStages]);
                    }
                }
                if (ab) {
                    if (lane == 0) bulk_wait_all();   // no store may still read this CTA's shared memory
                    return false;
                }
                pending = (long long)t;
                return true;
            });
        return;
    }
    // ------------------------------------------------------------------ consumers
    const unsigned ct = (unsigned)(tid - 96), nct = blockDim.x - 96;
    ring_tma_walk<DT>(P, r, n, c, ca, cb, SP, sent0, recvd0,
        [&](unsigned long long, int, int, bool) { return true; },
        [&](unsigned long long t, int s, unsigned long long, unsigned npk, unsigned long long, const uint4*, uint4*) {
            const int x = (int)(t % kRtStages);
            while (!mbar_try_wait(&full[x], (uint32_t)((t / kRtStages) & 1)))
                if (*(volatile int*)&s_abort) break;
            const bool ab = *(volatile int*)&s_abort != 0;
            if (!ab) {
                uint4* in = reinterpret_cast<uint4*>(in_smem(t));
                uint4* own = reinterpret_cast<uint4*>(own_smem(t));
                if (s == 0) {
                    if (AW > 1)
                        for (unsigned j = ct; j < npk; j += nct) {
                            Acc<DT> acc;
                            acc_init<DT>(acc, own[j]);
#pragma unroll
                            for (int y = 0; y < AW; ++y) in[j * AW + y] = acc.w[y];
                        }
                } else if (s < n) {
                    for (unsigned j = ct; j < npk; j += nct) {
                        Acc<DT> acc;
#pragma unroll
                        for (int y = 0; y < AW; ++y) acc.w[y] = in[j * AW + y];
                        acc_add<DT, OP>(acc, own[j]);
                        if (s < n - 1) {
#pragma unroll
                            for (int y = 0; y < AW; ++y) in[j * AW + y] = acc.w[y];
                        } else {
                            own[j] = acc_fin<DT>(acc);
                        }
                    }
                }
                if (s < n) fence_proxy_async_smem();   // my smem writes -> the bulk stores
            }
            __syncwarp();
            if (!ab && lane == 0) mbar_arrive(&cons[x]);
            return !ab;
        });
}

// ======================================================================= tree
// Binary tree per channel over positions pos = (rank - c) mod n (root = rank c
// mod n); children 2pos+1, 2pos+2.  Up phase: node = own (op) child0 (op)
// child1, partials (f32 for bf16) sent to the parent slot by slot; the root
// rounds once and stores.  Down phase: the result flows back down.

template <int PROTO>
__device__ __forceinline__ char* tree_base(const Params& P, int owner) {
    const unsigned long long off =
        PROTO == POLAR_PROTO_LL ? P.treell_off : PROTO == POLAR_PROTO_LL128 ? P.tree128_off : P.tree_off;
    return P.scratch[owner] + off;
}
template <int PROTO>
__device__ __forceinline__ uint4* tree_up_slot(const Params& P, int owner, int c, int child, unsigned long long seq) {
    return reinterpret_cast<uint4*>(tree_base<PROTO>(P, owner) +
                                    (((size_t)c * 2 + child) * kSteps + (seq % kSteps)) * tree_slot_bytes<PROTO>(P));
}
template <int PROTO>
__device__ __forceinline__ uint4* tree_dn_slot(const Params& P, int owner, int c, unsigned long long seq) {
    return reinterpret_cast<uint4*>(tree_base<PROTO>(P, owner) +
                                    ((size_t)kMaxCh * 2 * kSteps + (size_t)c * kSteps + (seq % kSteps)) *
                                        tree_slot_bytes<PROTO>(P));
}

template <int DT, int OP, int PROTO>
__device__ void tree(const Params& P, const Who& w) {
    constexpr int ES = DType<DT>::ES;
    constexpr int AW = AccWords<DT>::N;
    constexpr int U = batch_for<PROTO>() / AW > 0 ? batch_for<PROTO>() / AW : 1;
    using W = Wire<PROTO>;
    const int n = w.n, tid = w.tid, r = w.r, c = w.c;
    const int pos = ((r - c) % n + n) % n;
    auto rank_of = [&](int q) { return (q + c) % n; };
    const bool root = pos == 0;
    const int parent = root ? -1 : rank_of((pos - 1) / 2);
    const int my_child_idx = root ? 0 : (pos - 1) % 2;
    int child[2] = {-1, -1};
    int nchild = 0;
    for (int k = 0; k < 2; ++k)
        if (2 * pos + 1 + k < n) { child[k] = rank_of(2 * pos + 1 + k); nchild = k + 1; }

    ChanState* st = chan_state(P, r, c);
    unsigned long long usent = st->tree_usent, dsent = st->tree_dsent, drecv = st->tree_drecv;
    unsigned long long urecv[2] = {st->tree_urecv[0], st->tree_urecv[1]};
    const unsigned long long SP = W::units(tree_slot_bytes<PROTO>(P)) / AW * W::kPacks;
    const unsigned long long NP = npacks<ES>(P);
    unsigned long long ca, cb;
    split_range(0, NP, P.nch, c, ca, cb);
    const unsigned long long nslots = (cb - ca + SP - 1) / SP;
    char* mine = P.bufs[r];

    // ---------------------------------------------------------------- up
    for (unsigned long long s = 0; s < nslots; ++s) {
        const unsigned long long lo = ca + s * SP, hi = (lo + SP < cb) ? lo + SP : cb;
        bool ok = true;
        // thread k waits for child k's fill, thread 2 for the parent's credit.
        // Simple tails count HALF slots (2 per slot), the unit of tree_simple_ws,
        // which runs the same FIFOs for larger calls
        if (PROTO == POLAR_PROTO_SIMPLE && tid < nchild)
            ok = wait_geq(P, flag_ptr(P, r, F_TREE_UTAIL, c, tid), 2 * (urecv[tid] + 1));
        if (tid == 2 && !root && usent >= (unsigned long long)kSteps)
            ok = wait_geq(P, flag_ptr(P, r, F_TREE_UHEAD, c, 0), usent - kSteps + 1);
        if (!__syncthreads_and(ok)) return;
        uint4* dst = root ? nullptr : tree_up_slot<PROTO>(P, parent, c, my_child_idx, usent);
        const uint64_t fout = usent + 1;
        ok = for_batch<PROTO, U>(lo, hi, [&](const Batch<U>& b) {
            uint4 own[U];
            load_batch<ES>(P, mine, b, own);
            Acc<DT> acc[U];
#pragma unroll
            for (int u = 0; u < U; ++u) acc_init<DT>(acc[u], own[u]);
            if (PROTO == POLAR_PROTO_LL) {
                // LL: one child at a time (the joint poll holds 2x the raw lines;
                // measured 3-8 % slower)
                for (int k = 0; k < nchild; ++k) {
                    uint4 in[U][AW];
                    if (!get_batch<PROTO, U, AW>(P, tree_up_slot<PROTO>(P, r, c, k, urecv[k]), b, urecv[k] + 1, in))
                        return false;
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        Acc<DT> ch;
#pragma unroll
                        for (int q = 0; q < AW; ++q) ch.w[q] = in[u][q];
                        if (b.in[u]) acc_merge<DT, OP>(acc[u], ch);
                    }
                }
            } else if (nchild) {
                // both children's slots polled together (one wait, not two;
                // tree Simple 128 MiB 1576 -> 1409 us, LL128 2041 -> 1921 us)
                const uint4* src[2] = {tree_up_slot<PROTO>(P, r, c, 0, urecv[0]),
                                       tree_up_slot<PROTO>(P, r, c, 1, urecv[1])};
                const uint64_t fl[2] = {urecv[0] + 1, urecv[1] + 1};
                uint4 in[2][U][AW];
                if (!get_batch_multi<PROTO, 2, U, AW>(P, src, nchild, b, fl, in)) return false;
#pragma unroll
                for (int k = 0; k < 2; ++k)
                    if (k < nchild)
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            Acc<DT> ch;
#pragma unroll
                            for (int q = 0; q < AW; ++q) ch.w[q] = in[k][u][q];
                            if (b.in[u]) acc_merge<DT, OP>(acc[u], ch);
                        }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (!b.in[u]) continue;
                if (root) {
                    if (b.act[u]) store_pack<ES>(P, mine, b.i[u], acc_fin<DT>(acc[u]));
                } else {
#pragma unroll
                    for (int q = 0; q < AW; ++q) W::put(P, dst, b.j[u] * AW + q, acc[u].w[q], fout);
                }
            }
            return true;
        });
        if (!__syncthreads_and(ok)) return;
        if (PROTO == POLAR_PROTO_SIMPLE && POLAR_DISCARD && nchild) {
            for (int k = 0; k < nchild; ++k)
                discard_l2(tree_up_slot<PROTO>(P, r, c, k, urecv[k]), (hi - lo) * (unsigned long long)AW * 16ull);
            __syncthreads();
        }
        if (tid == 0) {
            if (PROTO == POLAR_PROTO_SIMPLE && (!root || (POLAR_DISCARD && nchild))) fence_acq_rel(P.sys);
            if (!root && PROTO == POLAR_PROTO_SIMPLE)
                jitter(P), st_relaxed(flag_ptr(P, parent, F_TREE_UTAIL, c, my_child_idx), 2 * (usent + 1), P.sys);
            for (int k = 0; k < nchild; ++k) jitter(P), st_relaxed(flag_ptr(P, child[k], F_TREE_UHEAD, c, 0), urecv[k] + 1, P.sys);
        }
        if (!root) ++usent;
        for (int k = 0; k < nchild; ++k) ++urecv[k];
    }
    // -------------------------------------------------------------- down
    for (unsigned long long s = 0; s < nslots; ++s) {
        const unsigned long long lo = ca + s * SP, hi = (lo + SP < cb) ? lo + SP : cb;
        bool ok = true;
        // thread 0: the parent's fill; threads 1, 2: the children's credits
        if (tid == 0 && !root && PROTO == POLAR_PROTO_SIMPLE) ok = wait_geq(P, flag_ptr(P, r, F_TREE_DTAIL, c, 0), 2 * (drecv + 1));
        if (tid >= 1 && tid <= nchild && dsent >= (unsigned long long)kSteps)
            ok = wait_geq(P, flag_ptr(P, r, F_TREE_DHEAD, c, tid - 1), dsent - kSteps + 1);
        if (!__syncthreads_and(ok)) return;
        const uint4* src = root ? nullptr : tree_dn_slot<PROTO>(P, r, c, drecv);
        const uint64_t fin = drecv + 1, fout = dsent + 1;
        ok = for_batch<PROTO, U>(lo, hi, [&](const Batch<U>& b) {
            uint4 v[U][1];
            if (root) {
                uint4 own[U];
                load_batch<ES>(P, mine, b, own);
#pragma unroll
                for (int u = 0; u < U; ++u) v[u][0] = own[u];
            } else {
                if (!get_batch<PROTO, U, 1>(P, src, b, fin, v)) return false;
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (b.act[u]) store_pack<ES>(P, mine, b.i[u], v[u][0]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (b.in[u])
                    for (int k = 0; k < nchild; ++k) W::put(P, tree_dn_slot<PROTO>(P, child[k], c, dsent), b.j[u], v[u][0], fout);
            return true;
        });
        if (!__syncthreads_and(ok)) return;
        if (PROTO == POLAR_PROTO_SIMPLE && POLAR_DISCARD && !root) {
            discard_l2(src, (hi - lo) * 16ull);
            __syncthreads();
        }
        if (tid == 0) {
            if (PROTO == POLAR_PROTO_SIMPLE && (nchild || (POLAR_DISCARD && !root))) fence_acq_rel(P.sys);
            if (PROTO == POLAR_PROTO_SIMPLE && nchild)
                for (int k = 0; k < nchild; ++k) jitter(P), st_relaxed(flag_ptr(P, child[k], F_TREE_DTAIL, c, 0), 2 * (dsent + 1), P.sys);
            if (!root) jitter(P), st_relaxed(flag_ptr(P, parent, F_TREE_DHEAD, c, my_child_idx), drecv + 1, P.sys);
        }
        if (nchild) ++dsent;
        if (!root) ++drecv;
    }
    if (tid == 0) {
        st->tree_usent = usent;
        st->tree_urecv[0] = urecv[0];
        st->tree_urecv[1] = urecv[1];
        st->tree_dsent = dsent;
        st->tree_drecv = drecv;
    }
}

// Tree Simple, warp specialised (POLAR_TREE_WS): the ring's scheme
// (ring_simple_ws) applied to both tree phases.  Units = half or whole slots; the sync
// warp's lanes 0..2 poll the unit's fills (children up / parent down) and
// credits (parent up / children down) in parallel, hand the unit over with
// READY, and publish the previous unit (fence, tails, credits after a slot's
// last unit) once its DONE completes.  At the up -> down boundary the last up
// unit is published BEFORE the first down wait: the parent's down phase needs it.
#ifndef POLAR_TREE_WS
#define POLAR_TREE_WS 1
#endif

template <int DT, int OP, int RQ>
__device__ void tree_simple_ws_impl(const Params& P, const Who& w) {
    constexpr int ES = DType<DT>::ES;
    constexpr int AW = AccWords<DT>::N;
    constexpr int U = POLAR_RING_WS_BATCH / AW > 0 ? POLAR_RING_WS_BATCH / AW : 1;
    constexpr int kReady = 1, kDone = 3;
    using W = Wire<POLAR_PROTO_SIMPLE>;
    const int n = w.n, tid = w.tid, r = w.r, c = w.c;
    const int nthr = blockDim.x;
    const int pos = ((r - c) % n + n) % n;
    auto rank_of = [&](int q) { return (q + c) % n; };
    const bool root = pos == 0;
    const int parent = root ? -1 : rank_of((pos - 1) / 2);
    const int my_child_idx = root ? 0 : (pos - 1) % 2;
    int child[2] = {-1, -1};
    int nchild = 0;
    for (int k = 0; k < 2; ++k)
        if (2 * pos + 1 + k < n) { child[k] = rank_of(2 * pos + 1 + k); nchild = k + 1; }
    ChanState* st = chan_state(P, r, c);
    unsigned long long usent = st->tree_usent, dsent = st->tree_dsent, drecv = st->tree_drecv;
    unsigned long long urecv[2] = {st->tree_urecv[0], st->tree_urecv[1]};
    const unsigned long long SP = W::units(P.tree_slot) / AW;   // element packs per slot
    const unsigned long long NP = npacks<ES>(P);
    unsigned long long ca, cb;
    split_range(0, NP, P.nch, c, ca, cb);
    const unsigned long long nslots = (cb - ca + SP - 1) / SP;
    // Units per slot (RQ, chosen by tree_simple_ws).  The tree is acyclic (a child's publication never waits on
    // its parent's current unit), so whole slots (RQ = 1) are valid here, unlike
    // in the ring.  Measured (profiles/r01_tree_ws_ab.jsonl): half slots pipeline
    // the levels when a channel has few slots (1 MiB 35.3 -> 29.7 us), whole slots
    // win at many slots (128 MiB 1176 -> 1066 us) and for tiny messages (4 KiB
    // 22.3 -> 19.0 us: fewer hand-offs).  Tail values count HALF slots whatever
    // RQ is, so flags stay monotone across calls that choose differently.
    constexpr unsigned long long QS = 2 / RQ;   // half slots per unit
    char* mine = P.bufs[r];
    __shared__ int s_abort;
    if (tid == 0) s_abort = 0;
    __syncthreads();

    if (tid < 32) {
        // ---------------------------------------------------------- sync warp
        const int lane = tid;
        unsigned long long g = 0;
        bool pending = false;
        uint64_t* pub_ptr[3] = {nullptr, nullptr, nullptr};   // unit g-1's flag stores
        uint64_t pub_val[3] = {0, 0, 0};
        int npub = 0;
        auto publish = [&]() {
            nbar_sync(kDone + (int)((g - 1) & 1), nthr);
            if (lane == 0) {
                fence_acq_rel(P.sys);
                for (int x = 0; x < npub; ++x) jitter(P), st_relaxed(pub_ptr[x], pub_val[x], P.sys);
            }
            pending = false;
        };
        for (int phase = 0; phase < 2; ++phase) {
            if (phase == 1 && pending) publish();   // the parent's down phase needs our last up unit
            for (unsigned long long sl = 0; sl < nslots; ++sl) {
                for (int q = 0; q < RQ; ++q) {
                    // lanes 0, 1: fills (up: child k; down: lane 0 the parent);
                    // lane 2 (up) / lanes 1, 2 (down): credits
                    int ok = 1;
                    if (phase == 0) {
                        if (lane < nchild) ok = wait_geq(P, flag_ptr(P, r, F_TREE_UTAIL, c, lane), urecv[lane] * 2 + (q + 1) * QS);
                        if (lane == 2 && q == 0 && !root && usent >= (unsigned long long)kSteps)
                            ok = wait_geq(P, flag_ptr(P, r, F_TREE_UHEAD, c, 0), usent - kSteps + 1);
                    } else {
                        if (lane == 0 && !root) ok = wait_geq(P, flag_ptr(P, r, F_TREE_DTAIL, c, 0), drecv * 2 + (q + 1) * QS);
                        if (lane >= 1 && lane <= nchild && q == 0 && dsent >= (unsigned long long)kSteps)
                            ok = wait_geq(P, flag_ptr(P, r, F_TREE_DHEAD, c, lane - 1), dsent - kSteps + 1);
                    }
                    ok = __all_sync(0xffffffffu, ok);
                    if (!ok && lane == 0) *(volatile int*)&s_abort = 1;
                    __syncwarp();
                    nbar_arrive(kReady + (int)(g & 1), nthr);
                    if (!ok) return;
                    if (pending) publish();
                    if (POLAR_WS_PREFETCH && phase == 0 && q == 0 && lane == 0 && sl + 1 < nslots) {
                        const unsigned long long a2 = ca + (sl + 1) * SP;   // own range of the next up slot
                        prefetch_own(P, mine, a2, (a2 + SP < cb) ? a2 + SP : cb, P.count * (unsigned long long)ES / 16);
                    }
                    npub = 0;
                    const bool last = q == RQ - 1;
                    if (phase == 0) {
                        if (!root) {
                            pub_ptr[npub] = flag_ptr(P, parent, F_TREE_UTAIL, c, my_child_idx);
                            pub_val[npub++] = usent * 2 + (q + 1) * QS;
                        }
                        if (last)
                            for (int k = 0; k < nchild; ++k) {
                                pub_ptr[npub] = flag_ptr(P, child[k], F_TREE_UHEAD, c, 0);
                                pub_val[npub++] = urecv[k] + 1;
                            }
                    } else {
                        for (int k = 0; k < nchild; ++k) {
                            pub_ptr[npub] = flag_ptr(P, child[k], F_TREE_DTAIL, c, 0);
                            pub_val[npub++] = dsent * 2 + (q + 1) * QS;
                        }
                        if (last && !root) {
                            pub_ptr[npub] = flag_ptr(P, parent, F_TREE_DHEAD, c, my_child_idx);
                            pub_val[npub++] = drecv + 1;
                        }
                    }
                    pending = true;
                    ++g;
                }
                if (phase == 0) {
                    if (!root) ++usent;
                    for (int k = 0; k < nchild; ++k) ++urecv[k];
                } else {
                    if (nchild) ++dsent;
                    if (!root) ++drecv;
                }
            }
        }
        if (pending) publish();
        if (lane == 0) {
            st->tree_usent = usent;
            st->tree_urecv[0] = urecv[0];
            st->tree_urecv[1] = urecv[1];
            st->tree_dsent = dsent;
            st->tree_drecv = drecv;
        }
        return;
    }
    // -------------------------------------------------------------- data warps
    const unsigned long long D = (unsigned long long)(nthr - 32), dt = (unsigned long long)(tid - 32);
    unsigned long long g = 0;
    for (int phase = 0; phase < 2; ++phase) {
        for (unsigned long long sl = 0; sl < nslots; ++sl) {
            const unsigned long long lo = ca + sl * SP, hi = (lo + SP < cb) ? lo + SP : cb;
            for (int q = 0; q < RQ; ++q) {
                const unsigned long long qs = lo + (hi - lo) * (unsigned long long)q / RQ;
                const unsigned long long qe = lo + (hi - lo) * (unsigned long long)(q + 1) / RQ;
                nbar_sync(kReady + (int)(g & 1), nthr);
                if (*(volatile int*)&s_abort) return;
                for (unsigned long long i0 = qs + dt; i0 < qe; i0 += U * D) {
                    Batch<U> b;
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        b.i[u] = i0 + u * D;
                        b.j[u] = b.i[u] - lo;               // wire index in the slot
                        b.in[u] = b.act[u] = b.i[u] < qe;
                    }
                    if (phase == 0) {
                        uint4 own[U];
                        load_batch<ES>(P, mine, b, own);
                        uint4 in[2][U][AW];
#pragma unroll
                        for (int k = 0; k < 2; ++k)
                            if (k < nchild) {
                                const uint4* src = tree_up_slot<POLAR_PROTO_SIMPLE>(P, r, c, k, urecv[k]);
#pragma unroll
                                for (int u = 0; u < U; ++u)
#pragma unroll
                                    for (int x = 0; x < AW; ++x)
                                        if (b.in[u]) in[k][u][x] = ld_cg(src + b.j[u] * AW + x);
                            }
                        uint4* dst = root ? nullptr : tree_up_slot<POLAR_PROTO_SIMPLE>(P, parent, c, my_child_idx, usent);
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            if (!b.in[u]) continue;
                            Acc<DT> acc;
                            acc_init<DT>(acc, own[u]);
#pragma unroll
                            for (int k = 0; k < 2; ++k)
                                if (k < nchild) {
                                    Acc<DT> ch;
#pragma unroll
                                    for (int x = 0; x < AW; ++x) ch.w[x] = in[k][u][x];
                                    acc_merge<DT, OP>(acc, ch);
                                }
                            if (root) store_pack<ES>(P, mine, b.i[u], acc_fin<DT>(acc));
                            else
#pragma unroll
                                for (int x = 0; x < AW; ++x) W::put(P, dst, b.j[u] * AW + x, acc.w[x], 0);
                        }
                    } else {
                        uint4 v[U];
                        if (root) {
                            load_batch<ES>(P, mine, b, v);
                        } else {
                            const uint4* src = tree_dn_slot<POLAR_PROTO_SIMPLE>(P, r, c, drecv);
#pragma unroll
                            for (int u = 0; u < U; ++u)
                                if (b.in[u]) v[u] = ld_cg(src + b.j[u]);
#pragma unroll
                            for (int u = 0; u < U; ++u)
                                if (b.in[u]) store_pack<ES>(P, mine, b.i[u], v[u]);
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u)
                            if (b.in[u])
                                for (int k = 0; k < nchild; ++k)
                                    W::put(P, tree_dn_slot<POLAR_PROTO_SIMPLE>(P, child[k], c, dsent), b.j[u], v[u], 0);
                    }
                }
                nbar_arrive(kDone + (int)(g & 1), nthr);
                ++g;
            }
            if (phase == 0) {
                if (!root) ++usent;
                for (int k = 0; k < nchild; ++k) ++urecv[k];
            } else {
                if (nchild) ++dsent;
                if (!root) ++drecv;
            }
        }
    }
}

#ifndef POLAR_TREE_WS_MIN
#define POLAR_TREE_WS_MIN 16384   // bytes per channel below which tree Simple runs the plain kernel
#endif
template <int DT, int OP>
__device__ void tree_simple_ws(const Params& P, const Who& w) {
    constexpr int ES = DType<DT>::ES;
    constexpr int AW = AccWords<DT>::N;
    unsigned long long ca, cb;
    split_range(0, npacks<ES>(P), P.nch, w.c, ca, cb);
    const unsigned long long SP = Wire<POLAR_PROTO_SIMPLE>::units(P.tree_slot) / AW;
    // the same on every rank of a channel (ca, cb depend only on the channel).
    // Below 16 KiB per channel the plain tree (one slot, no hand-offs) is faster
    // (4-64 KiB: 17.7 vs 19.7-20.1 us); its Simple tails count half slots too
    const unsigned long long bytes = (cb - ca) * 16ull;
    if (bytes < POLAR_TREE_WS_MIN) tree<DT, OP, POLAR_PROTO_SIMPLE>(P, w);
    else if ((cb - ca + SP - 1) / SP <= 4) tree_simple_ws_impl<DT, OP, 2>(P, w);
    else tree_simple_ws_impl<DT, OP, 1>(P, w);
}

// ============================================== cross-rank decision check
// SURVEY.md §8(b) "cross-rank consistency" (R12): on a real comm every
// rank decides locally, so ranks that disagree (a policy swapped on one rank
// only, different counts, ops or channel counts) would exchange mismatched data
// — silently wrong results or a timeout.  Each launch's thread 0 of CTA 0
//   tag_begin: publishes {call, tag} in its own scratch ring and issues
//              cp.async copies of every peer's entry for call - 1 into shared
//              memory (no registers held, the NVLink round trip overlaps the
//              collective);
//   tag_end:   waits for the copies and latches POLAR_ESTATE if a peer's entry
//              for call - 1 carries a different tag.
// Detection is one launch late and never a false positive: an entry whose call
// stamp is not call - 1 (not yet visible) is skipped.  Each 8-B half of the
// 16-B entry carries the call stamp ({tag_lo, call}, {tag_hi, call}), so a torn
// read is rejected, not misread.  Virtual comms decide once for all ranks.
__device__ __forceinline__ const char* tag_entry(const Params& P, int rank, unsigned long long call) {
    return P.scratch[rank] + P.tags_off + (call % kTagRing) * 16;
}
__device__ __forceinline__ void tag_begin(const Params& P, uint4* s_tags) {
    if (!P.sys || blockIdx.x != 0 || threadIdx.x != 0) return;
    const uint32_t c = (uint32_t)P.call;
    st_ll(reinterpret_cast<uint4*>(const_cast<char*>(tag_entry(P, P.rank0, P.call))), (uint32_t)P.dtag,
          (uint32_t)(P.dtag >> 32), c);
    if (P.call == 0) return;
    for (int p = 0; p < P.nranks; ++p)
        if (p != P.rank0)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&s_tags[p])),
                         "l"(tag_entry(P, p, P.call - 1))
                         : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tag_end(const Params& P, const uint4* s_tags) {
    if (!P.sys || blockIdx.x != 0 || threadIdx.x != 0 || P.call == 0) return;
    asm volatile("cp.async.wait_all;" ::: "memory");
    const uint32_t c = (uint32_t)(P.call - 1);
    for (int p = 0; p < P.nranks; ++p) {
        if (p == P.rank0) continue;
        const uint4 t = s_tags[p];
        if (t.y == c && t.w == c && (t.x | ((unsigned long long)t.z << 32)) != P.prev_tag) raise_error(P, POLAR_ESTATE);
    }
}

// ================================================================== kernels

template <int DT, int OP, int ALGO, int PROTO>
__global__ void __launch_bounds__(kBlock, POLAR_LB_MIN) allreduce_kernel(Params P) {
    // Programmatic dependent launch: let the NEXT polar launch on this stream get
    // its CTAs scheduled during our tail, and wait here until the previous grid
    // has completed and its memory is visible (== plain stream order; no-ops
    // when the launch carries no PDL attribute).
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __shared__ __align__(16) uint4 s_tags[kMaxRanks];
    tag_begin(P, s_tags);
    const Who w = who(P);
    // profiler telemetry (f3): CTA 0 stamps the launch into the host-mapped ring
    const bool tel = P.tel != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
    const unsigned long long tel_t0 = tel ? globaltimer() : 0;
    if constexpr (ALGO == POLAR_ALGO_TWOSHOT) {
        if constexpr (PROTO == POLAR_PROTO_SIMPLE) twoshot_simple<DT, OP>(P, w);
        else twoshot_ll<DT, OP, PROTO>(P, w);
    } else if constexpr (ALGO == POLAR_ALGO_ONESHOT) {
        if constexpr (PROTO == POLAR_PROTO_SIMPLE) oneshot_simple<DT, OP>(P, w);
        else oneshot_ll<DT, OP, PROTO>(P, w);
    } else if constexpr (ALGO == POLAR_ALGO_RING) {
        if constexpr (PROTO == POLAR_PROTO_SIMPLE && POLAR_RING_WS) {
            // TMA staging needs whole 16-B packs of a 16-B aligned buffer (uniform per launch)
            if (POLAR_RING_TMA && P.ring_tma && P.vec && (P.count * DType<DT>::ES) % 16 == 0)
                ring_simple_tma<DT, OP>(P, w);
            else
                ring_simple_ws<DT, OP>(P, w);
        } else {
            ring<DT, OP, PROTO>(P, w);
        }
    } else {
        if constexpr (PROTO == POLAR_PROTO_SIMPLE && POLAR_TREE_WS) tree_simple_ws<DT, OP>(P, w);
        else tree<DT, OP, PROTO>(P, w);
    }
    tag_end(P, s_tags);
    if (tel) {
        volatile TelEntry* e = P.tel + (P.seq % kTelRing);
        e->t0 = tel_t0;
        e->t1 = globaltimer();
        __threadfence_system();
        e->seq = P.seq;
    }
}


// ============================================================ direct collectives
// ReduceScatter / AllGather / Broadcast through the same hook (SURVEY.md §8(f)
// f4; oracle/collectives.py): one all-to-all step on peer-mapped symmetric
// buffers between the two-shot's entry and exit barriers.  P.count = elements
// per block (RS: recvcount, AG: sendcount, BC: count).
//   RS: owner r pulls block r from every rank's send buffer, reduces in rank
//       order, stores its receive buffer            (ingress (n-1)/n of the input)
//   AG: rank r pushes its block into block r of every rank's receive buffer
//   BC: every rank pulls root's buffer                (root only synchronises)
enum { MODE_RS = 0, MODE_AG = 1, MODE_BC = 2 };

template <int DT, int OP, int MODE>
__global__ void __launch_bounds__(kBlock, POLAR_LB_MIN) direct_kernel(Params P) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    constexpr int ES = DType<DT>::ES;
    __shared__ __align__(16) uint4 s_tags[kMaxRanks];
    tag_begin(P, s_tags);
    const Who w = who(P);
    const int n = w.n, tid = w.tid;
    ChanState* st = chan_state(P, w.r, w.c);
    const uint64_t e = st->epoch + 1;
    if (!handshake_entry(P, w, e)) return;
    const unsigned long long NP = npacks<ES>(P);
    const size_t blk_bytes = (size_t)P.count * ES;
    unsigned long long a, b;
    split_range(0, NP, P.nch, w.c, a, b);
    const unsigned long long stride = (unsigned long long)blockDim.x;
    if constexpr (MODE == MODE_RS) {
        // every rank's pack issued before the reduction (n loads in flight per thread)
        for (unsigned long long i = a + tid; i < b; i += stride) {
            uint4 v[kMaxRanks];
#pragma unroll
            for (int p = 0; p < kMaxRanks; ++p)
                if (p < n) v[p] = load_pack<ES>(P, P.bufs[p] + (size_t)w.r * blk_bytes, i);
            Acc<DT> acc;
            acc_init<DT>(acc, v[0]);
#pragma unroll
            for (int p = 1; p < kMaxRanks; ++p)
                if (p < n) acc_add<DT, OP>(acc, v[p]);
            store_pack<ES>(P, P.recv[w.r], i, acc_fin<DT>(acc));
        }
    } else if constexpr (MODE == MODE_AG) {
        constexpr int U = 1;   // (U = 4 measured slower: 454 vs 507 GB/s busBW at 256 MiB)
        for (unsigned long long i0 = a + tid; i0 < b; i0 += U * stride) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (i0 + u * stride < b) v[u] = load_pack<ES>(P, P.bufs[w.r], i0 + u * stride);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (i0 + u * stride < b) {
#pragma unroll
                    for (int p = 0; p < kMaxRanks; ++p)
                        if (p < n) store_pack<ES>(P, P.recv[p] + (size_t)w.r * blk_bytes, i0 + u * stride, v[u]);
                }
        }
    } else {
        // Broadcast: every non-root rank pulls the root's slice, 8 packs per thread
        // in flight.  (Staggering the ranks' pull order was measured slower: the
        // concurrent pulls of the same root lines are served from L2.)
        constexpr int U = 8;
        if (w.r != P.root)
            for (unsigned long long i0 = a + tid; i0 < b; i0 += U * stride) {
                uint4 v[U];
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (i0 + u * stride < b) v[u] = load_pack<ES>(P, P.bufs[P.root], i0 + u * stride);
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (i0 + u * stride < b) store_pack<ES>(P, P.bufs[w.r], i0 + u * stride, v[u]);
            }
    }
    __syncthreads();
    if (!handshake_exit(P, w, e)) return;
    epoch_publish(P, w, e);
    tag_end(P, s_tags);
}

}  // namespace dev
}  // namespace polar
