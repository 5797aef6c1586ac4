/*
 * polar.h — C ABI of libpolar, a policy-selected AllReduce for B200 (sm_100a).
 *
 * The hot path is: a bounded tuner decision keyed by
 * (collective, bytes, nranks) picks an algorithm, a protocol and a channel count
 * (§2, §3.3), then ONE hand-written sm_100a kernel
 * moves and reduces the data by reading/writing peer buffers directly
 * (NVLink/NVSwitch peer mappings on a real node; the same kernels drive
 * "virtual ranks" that share one GPU).
 *
 * Conventions for every function:
 *   - Nothing aborts, throws or exits across this ABI; every call returns a
 *     polar_status (or a plain value where documented).
 *   - "device pointer" = memory on the comm's CUDA device (cudaMalloc /
 *     torch); "host pointer" = ordinary process memory.
 *   - Streams are passed as `void*` holding a cudaStream_t (NULL = legacy
 *     default stream); kernels are enqueued asynchronously, no host sync.
 *   - Collective functions must be called by every rank of the comm, in the same
 *     order, with matching arguments (NCCL rules); one host thread per comm at a
 *     time.  Policy functions are process-global and thread-safe.
 *   - Errors raised on the device (a peer that never arrives) are latched in the
 *     comm and returned by the NEXT call on it, or by polar_comm_check().
 *   - Cross-rank consistency (the paper is silent, DESIGN.md
 *     R12): on a real comm every launch carries a decision tag (kind, algorithm,
 *     protocol, channels, dtype, op, count, root, and for zero-copy kernels the
 *     buffer path: registration id + offset, or the bounce region).
 *       * Kernels with an entry handshake (two-shot Simple, ReduceScatter,
 *         AllGather, Broadcast) exchange the tag inside it: ranks that disagree
 *         latch POLAR_ESTATE and leave BEFORE any data moves (synchronous).
 *       * Every other kernel publishes its tag in its scratch and compares its
 *         peers' tags of the PREVIOUS launch: a difference latches POLAR_ESTATE
 *         one launch late; the mismatched call's output is undefined, and the
 *         last call of a sequence is only checked by a following launch.
 *     Ranks that pick different kernels altogether (a policy swapped on one
 *     rank only) usually wait for each other in vain: POLAR_ETIMEOUT.
 *       * Under polar_comm_autoreg every call of >= min_bytes all-gathers the
 *         decision tag on the host first: a disagreement returns POLAR_ESTATE
 *         on every rank before anything is launched.
 */
#ifndef POLAR_H
#define POLAR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ enums */

typedef enum {
    POLAR_OK = 0,
    POLAR_EINVAL = 1,        /* malformed argument or policy table                   */
    POLAR_ECUDA = 2,         /* a CUDA runtime/driver call failed                     */
    POLAR_EUNSUPPORTED = 3,  /* well-formed but not built (NVLS; no kernel for a decision) */
    POLAR_ETIMEOUT = 4,      /* a device-side wait for a peer exceeded the timeout    */
    POLAR_EBUSY = 5,         /* concurrent use of a single-threaded object            */
    POLAR_ESTATE = 6,        /* comm unusable (earlier latched error / destroyed)     */
    POLAR_ENOMEM = 7         /* device or host allocation failed                      */
} polar_status;

/* dtype / op use NCCL's numbering so one harness can drive both (nccl.h). */
typedef enum { POLAR_INT32 = 2, POLAR_INT64 = 4, POLAR_FLOAT32 = 7, POLAR_BFLOAT16 = 9 } polar_dtype;
typedef enum { POLAR_SUM = 0, POLAR_MAX = 2, POLAR_MIN = 3 } polar_op;

/* Collective / algorithm / protocol enums: SPEC.md L306 numbering
 * (TREE=0, RING=1, NVLS=2; LL=0, LL128=1, SIMPLE=2) plus the two direct
 * all-to-all algorithms this library adds. */
enum { POLAR_COLL_ALLREDUCE = 0, POLAR_COLL_ALLGATHER = 1, POLAR_COLL_BROADCAST = 2,
       POLAR_COLL_REDUCESCATTER = 3 };
enum { POLAR_ALGO_TREE = 0, POLAR_ALGO_RING = 1, POLAR_ALGO_NVLS = 2 /* switch reduction, f1 */,
       POLAR_ALGO_ONESHOT = 3, POLAR_ALGO_TWOSHOT = 4 };
enum { POLAR_PROTO_LL = 0, POLAR_PROTO_LL128 = 1, POLAR_PROTO_SIMPLE = 2 };

#define POLAR_UNSET 0xFFFFFFFFu   /* algo/proto "defer to default"   */
#define POLAR_MAXCH 32            /* channel clamp bound (R8) */
#define POLAR_MAXRANKS 8          /* one NVLink node                                 */
#define POLAR_MAXROWS 64          /* bounded policy table                            */

/* ---------------------------------------------------------------- structs */

/* Tuner context ("collective type, message size, rank count"). 16 B. */
typedef struct {
    uint32_t coll;     /* POLAR_COLL_*                                     */
    uint32_t nranks;   /* participating ranks, 1..POLAR_MAXRANKS          */
    uint64_t bytes;    /* total message bytes = count * element size      */
} polar_ctx;

/* Tuner outputs ("writes algorithm, protocol, and channel count")
 * plus the policy generation that produced them and the
 * matching row's flags. 24 B. */
typedef struct {
    uint32_t algo;        /* POLAR_ALGO_*                                          */
    uint32_t proto;       /* POLAR_PROTO_*                                         */
    uint32_t nchannels;   /* 1..POLAR_MAXCH (with POLAR_ROW_ADAPTIVE_NCH: the cap) */
    uint32_t generation;  /* active policy generation at decide                    */
    uint32_t flags;       /* POLAR_ROW_* of the matching row (0 if none / default)  */
    uint32_t _pad;
} polar_decision;

/* Row flags.  POLAR_ROW_ADAPTIVE_NCH: the channel count is chosen per call by the
 * comm's profiler->tuner closed loop (polar_adaptive_*; PAPER.md L311-351,
 * L597-611), between the controller's c_min and this row's nchannels (the cap). */
#define POLAR_ROW_ADAPTIVE_NCH 0x1u

/* One policy row. 32 B.  A policy is an ordered list of rows; the first row with
 * coll == ctx.coll, nranks in {0 (any), ctx.nranks} and ctx.bytes <= max_bytes
 * (inclusive, "msg_size <= 32*1024") wins.  algo/proto may be
 * POLAR_UNSET and nchannels 0 to defer that field to the built-in default
 * (SPEC.md L339); nchannels is clamped to [1, POLAR_MAXCH]. */
typedef struct {
    uint32_t coll;
    uint32_t nranks;      /* 0 = any                                */
    uint64_t max_bytes;   /* inclusive upper bound on message bytes */
    uint32_t algo;        /* POLAR_ALGO_* or POLAR_UNSET            */
    uint32_t proto;       /* POLAR_PROTO_* or POLAR_UNSET           */
    uint32_t nchannels;   /* 0 = UNSET; any other u32 is clamped    */
    uint32_t flags;       /* POLAR_ROW_* bits; others must be 0     */
} polar_policy_row;

/* Host all-gather (comm init, registration, collective barriers, and once per
 * call of >= min_bytes under polar_comm_autoreg): gathers bytes_per_rank from
 * every rank into recv (rank order); every rank passes the same size in one
 * call.  Return 0 on success. */
typedef int (*polar_allgather_fn)(const void* send, void* recv, size_t bytes_per_rank, void* user);

typedef struct polar_comm_s* polar_comm_t;   /* opaque; owned by the library */

/* ------------------------------------------------------ policy (decision hook) */

/* Atomically replace the process-global policy (§4 "atomic
 * compare-and-swap on the pointer").  The rows are COPIED.
 * Validation: nrows <= 64; known enums; nranks <= 8; only known flag bits; rows of one
 * (coll, nranks) group strictly ascending in max_bytes -> else POLAR_EINVAL;
 * a decision no kernel implements -> POLAR_EUNSUPPORTED: NVLS while no comm of
 * this process holds a multicast object (polar_nvls_available), and
 * ReduceScatter / AllGather / Broadcast rows naming anything but ONESHOT /
 * SIMPLE (or UNSET).  LL128 is accepted (every AllReduce algorithm has an
 * LL128 kernel; real comms refuse it at call time
 * until the line-atomicity probe passed over their transport, see
 * polar_allreduce).  On any rejection the active policy and
 * its generation are unchanged ("the old policy continues").
 * nrows == 0 installs the empty policy (the paper's `noop`, L433).
 * On success the generation increases by exactly 1 and is stored in
 * *generation_out (may be NULL).  Retired tables stay allocated until process
 * exit, so in-flight polar_decide calls never read freed memory (drain safety). */
polar_status polar_set_policy(const polar_policy_row* rows, uint32_t nrows, uint32_t* generation_out);

/* The decision hook: pure, wait-free (one acquire load + a <=64-row scan), any
 * thread.  UNSET fields defer to the built-in default table (DESIGN.md "Default
 * table"); nchannels clamped to [1, POLAR_MAXCH].  A collective without a
 * default row (unknown coll) -> POLAR_EUNSUPPORTED; NULL pointers or nranks
 * outside 1..8 -> POLAR_EINVAL. */
polar_status polar_decide(const polar_ctx* ctx, polar_decision* out);

/* Batched form for sweeps/tests: out[i] = decide(ctx[i]); stops at the first error. */
polar_status polar_decide_batch(const polar_ctx* ctx, polar_decision* out, size_t n);

/* Active generation (0 before the first successful polar_set_policy). */
uint32_t polar_policy_generation(void);

/* Copy out the active rows (cap entries at most) and generation. */
polar_status polar_get_policy(polar_policy_row* rows, uint32_t cap, uint32_t* nrows, uint32_t* generation);

/* ------------------------------------------------------- decision-cost bench */

typedef struct {
    uint64_t calls;             /* timed calls                                   */
    double p50_ns, p99_ns;      /* per-call, raw (timer pair included)           */
    double mean_ns, min_ns, max_ns;
    double timer_overhead_ns;   /* p50 of an empty timer pair                    */
    double batched_mean_ns;     /* total / calls of an untimed-per-call loop      */
} polar_bench_stats;

/* BASELINE.json config 5 (SPEC.md L477-481 method): nwarm untimed warm-up calls,
 * then ncalls calls each timed with a monotonic clock into a full sample buffer
 * (samples_ns may be NULL; else ncalls entries), cycling through ctxs[0..nctx). */
polar_status polar_bench_decide(const polar_ctx* ctxs, uint32_t nctx, uint64_t nwarm, uint64_t ncalls,
                                uint64_t* samples_ns, polar_bench_stats* out);

typedef struct {
    uint64_t calls;             /* decisions returned (must equal issued)        */
    uint64_t issued;            /* decisions requested                           */
    uint64_t invalid;           /* decisions not produced by their generation's table */
    uint64_t nonmonotonic;      /* per-thread generation decreases               */
    uint64_t swaps;             /* successful swaps                              */
    uint64_t rejected;          /* rejected (invalid-table) reload attempts      */
    uint64_t rejected_changed;  /* rejections that changed the generation (must be 0) */
    double swap_p50_ns, swap_p99_ns, swap_max_ns;   /* duration of the pointer swap */
    uint32_t final_generation;
} polar_swap_stats;

/* SPEC.md L444-446 zero-loss stress: nthreads invokers issue calls_per_thread
 * decisions each while one reloader alternates tables A and B nswaps times and,
 * every 10th swap, attempts an invalid table that must be rejected.  Leaves
 * the last installed table active. */
polar_status polar_bench_swap(uint32_t nthreads, uint64_t calls_per_thread, uint32_t nswaps,
                              const polar_policy_row* a, uint32_t na,
                              const polar_policy_row* b, uint32_t nb,
                              polar_swap_stats* out);

/* ------------------------------------------------------------ communicators */

/* Real multi-process comm: one rank per process, one GPU per rank (SURVEY.md
 * §3(4)).  Allocates this rank's symmetric scratch (flags + staging) on
 * cuda_device, exchanges CUDA IPC handles through `ag` (the only host
 * collective), maps every peer's scratch and runs a device handshake.
 * Collective.  nranks 1..8, 0 <= rank < nranks.  Ranks that share one GPU
 * (several processes per device, e.g. under MPS) are detected from the GPU
 * UUIDs: programmatic dependent launch is then off, and every launch's channel
 * count is capped at the device's co-resident CTAs / the ranks per GPU (the
 * minimum over ranks), so that every rank's CTAs can be resident together —
 * polar_comm_last_decision still reports the policy's decision,
 * polar_comm_launch_info what was launched.  One rank per GPU: no cap. */
polar_status polar_comm_init(polar_comm_t* out, int nranks, int rank, int cuda_device,
                             polar_allgather_fn ag, void* user);

/* Host bootstrap self-check (collective; no GPU needed): all-gathers a 32-B
 * record {magic, nranks, rank, scratch-layout hash} through `ag` and verifies
 * that every rank agrees on nranks and on the scratch layout (the POLAR_* size
 * variables) and that slot p holds rank p.  POLAR_OK, POLAR_EINVAL (bad args),
 * or POLAR_ESTATE (disagreement or callback failure).  polar_comm_init runs the
 * same check before it exchanges any IPC handle. */
polar_status polar_bootstrap_check(int nranks, int rank, polar_allgather_fn ag, void* user);

/* Virtual comm: nranks logical ranks hosted by THIS process on ONE device; one
 * kernel launch runs every rank's CTAs (grid = nranks x nchannels, clamped to
 * the device's co-resident CTA count so that cross-rank waits cannot deadlock
 * on an otherwise idle GPU; plain launch + programmatic dependent launch like
 * real comms, POLAR_VIRTUAL_COOP=1 forces a cooperative launch).  Same kernels,
 * same protocols; peers are local HBM instead of NVLink (DESIGN.md "Virtual
 * ranks").  Every cross-rank wait is bounded (POLAR_TIMEOUT_MS).
 * Concurrency: the launch is plain (not cooperative), sized so that every CTA
 * is resident on an otherwise idle GPU.  Keep ONE virtual-comm collective in
 * flight per device at a time: two concurrent grids (two virtual comms, or one
 * comm on two streams) can each hold SMs the other's spinning CTAs need, which
 * ends in POLAR_ETIMEOUT (latched) instead of a result.  POLAR_VIRTUAL_COOP=1
 * makes the launch cooperative (co-residency checked by the runtime, ~2 us more
 * per call). */
polar_status polar_comm_init_virtual(polar_comm_t* out, int nranks, int cuda_device);

/* Collective for real comms: synchronises the device, host-barriers through the
 * all-gather (no peer still touches this rank's memory), then unmaps and frees. */
polar_status polar_comm_destroy(polar_comm_t comm);

/* nranks, this process's first rank, and how many ranks this process hosts
 * (1 for a real comm, nranks for a virtual one).  Any out pointer may be NULL. */
polar_status polar_comm_info(polar_comm_t comm, int* nranks, int* rank, int* nlocal);

/* Symmetric allocation (collective): `bytes` of device memory per local rank,
 * peer-mapped on every rank, so AllReduce on it is zero-copy.  ptrs receives
 * nlocal device pointers.  Freed by polar_mem_free (collective) or destroy. */
polar_status polar_mem_alloc(polar_comm_t comm, size_t bytes, void** ptrs);
/* Collective for real comms (barrier, unmap the peers' copies, barrier, free). */
polar_status polar_mem_free(polar_comm_t comm, void* ptr);

/* Register caller-owned device memory [buf, buf+bytes) for zero-copy use
 * (collective; every rank registers its own buffer in the same call order).
 * Virtual comms accept and ignore it (all ranks are local).  A registration
 * remembers its allocation (CU_POINTER_ATTRIBUTE_BUFFER_ID): once that
 * allocation is freed (cudaFree; a caching allocator that keeps the segment
 * does not free it) the registration is stale and is dropped at its next use,
 * and the call takes the unregistered path — if another rank still uses its
 * registration for the same call, the entry handshake latches POLAR_ESTATE. */
polar_status polar_register(polar_comm_t comm, void* buf, size_t bytes);

/* Drop the registration whose start is `buf` (collective: synchronises the
 * device, host-barriers, closes the peers' IPC mappings no other registration
 * uses).  POLAR_OK also when `buf` is not (or no longer) registered. */
polar_status polar_deregister(polar_comm_t comm, void* buf);

/* Auto-registration (collective; every rank passes the same values, else
 * POLAR_EINVAL and nothing changes).  With enable != 0, every real-comm
 * AllReduce of >= min_bytes exchanges, through the comm's all-gather callback,
 * each rank's {decision tag, CUDA-IPC handle of the allocation holding the
 * buffer, its buffer id, the buffer's offset} — whatever the rank's decision or
 * registrations, so the exchanges line up on every rank; ranks that decided the
 * call differently all return (and latch) POLAR_ESTATE here, synchronously,
 * before anything is launched.  When the decision is two-shot Simple each rank
 * maps the peers' allocations (opened once per
 * allocation and cached, at most 32 per peer, least recently used closed after a
 * device synchronise) and the call runs zero-copy, as on a registration.  So the
 * call costs one small host all-gather instead of the bounce region's local
 * copies (north_star's allreduce(buf, ...) on caller memory).
 * Offsets may differ between ranks, and registrations are not consulted.  If
 * any rank's buffer is not IPC-exportable (cuMem/VMM memory, e.g. expandable
 * segments) every rank takes the bounce path for that call — the choice
 * depends on the gathered records only, so ranks agree.  No mapping is closed
 * while the caller's stream is being captured (the cache may then exceed its
 * bound).  A peer allocation freed and re-allocated is detected
 * by its buffer id (the stale mapping is closed and the new one opened).  The
 * all-gather callback is invoked from inside polar_allreduce (also while a
 * stream is being captured into a CUDA graph: the graph keeps the pointers of
 * capture time).  Virtual comms accept and ignore it.  Default: off. */
polar_status polar_comm_autoreg(polar_comm_t comm, int enable, size_t min_bytes);

typedef struct {
    uint64_t exchanges;  /* auto-registration exchanges (one host all-gather each) */
    uint64_t zero_copy;  /* ... of which ran zero-copy */
    uint64_t bounced;    /* ... of which took the bounce path (a rank's buffer not exportable) */
    uint64_t opens;      /* peer allocations opened (cudaIpcOpenMemHandle) */
    uint64_t evictions;  /* auto-opened mappings closed (cache bound, stale allocation) */
    uint64_t mismatches; /* exchanges whose ranks had decided the call differently (ESTATE) */
} polar_autoreg_stats;
polar_status polar_comm_autoreg_stats(polar_comm_t comm, polar_autoreg_stats* out);

/* ----------------------------------------------------------------- AllReduce */

/* In-place AllReduce of `count` elements at device pointer `buf` (real comm,
 * nlocal == 1).  Decides (hook above), then launches ONE kernel on `stream`.
 * count == 0 or nranks == 1 -> POLAR_OK without a launch.  buf need not be
 * 16-B aligned (a scalar path is used) nor registered: an unregistered buffer
 * under two-shot travels through the symmetric bounce region (POLAR_BOUNCE,
 * default 2 x 32 MiB) in chunks whose copy-in (library stream), kernel (this
 * stream) and copy-out (library stream) overlap; `stream` waits for the last
 * copy-out.  NULL buf with count > 0, bad dtype/op -> POLAR_EINVAL; an LL128
 * decision before polar_comm_probe_ll128 passed, or NVLS without a multicast
 * object -> POLAR_EUNSUPPORTED.  Result: every rank holds the rank-ordered reduction
 * (SURVEY.md §8(c)), bitwise identical on every rank. */
polar_status polar_allreduce(polar_comm_t comm, void* buf, size_t count, polar_dtype dtype,
                             polar_op op, void* stream);

/* Same, for any comm: bufs[nlocal] device pointers, one per local rank
 * (virtual comms: rank r's buffer is bufs[r]). */
polar_status polar_allreduce_v(polar_comm_t comm, void* const* bufs, size_t count, polar_dtype dtype,
                               polar_op op, void* stream);

/* Same, but the decision is forced (sweeps, BASELINE config 3); `forced`'s
 * algo/proto must be concrete, nchannels is clamped; generation is ignored. */
polar_status polar_allreduce_forced(polar_comm_t comm, void* const* bufs, size_t count,
                                    polar_dtype dtype, polar_op op, const polar_decision* forced,
                                    void* stream);

/* End-to-end form over HOST memory: host_bufs[nlocal] (pinned for overlap;
 * pageable works but serialises) are copied to the device buffers
 * dev_bufs[nlocal], reduced in place, and the result is copied back into
 * host_bufs; synchronous (returns after the last D2H copy completed).  The
 * message is processed in chunks of POLAR_HOST_CHUNK bytes per rank (default
 * 8 MiB): the H2D copy of chunk k+1, the AllReduce of chunk k (one decision and
 * one launch per chunk, on `stream`) and the D2H copy of chunk k-1 overlap on
 * two library-owned copy streams.  Chunking does not change the result (the
 * reduction is elementwise).  Used for the bench's e2e number. */
polar_status polar_allreduce_host(polar_comm_t comm, void* const* host_bufs, void* const* dev_bufs,
                                  size_t count, polar_dtype dtype, polar_op op, void* stream);

/* Host enqueue cost (BASELINE config 4 "host enqueue ns per call"): ncalls
 * back-to-back polar_allreduce_v calls (decide + dispatch + launch, no sync)
 * timed with a monotonic clock; *ns_per_call = wall time / ncalls.  The stream
 * is synchronised before and after the timed loop. */
polar_status polar_bench_enqueue(polar_comm_t comm, void* const* bufs, size_t count, polar_dtype dtype,
                                 polar_op op, void* stream, uint64_t ncalls, double* ns_per_call);

/* ------------------------------------------ other collectives through the hook (f4)
 * ReduceScatter, AllGather and Broadcast are decided by the same hook
 * (ctx.coll = POLAR_COLL_REDUCESCATTER / ALLGATHER / BROADCAST; ctx.bytes = the
 * full buffer: recvcount*n*esize, sendcount*n*esize, count*esize) and run as ONE
 * direct all-to-all step between an entry and an exit barrier (only algo
 * ONESHOT + proto SIMPLE exist for them; any other decision -> EUNSUPPORTED).
 * Semantics (NCCL's; oracle/collectives.py):
 *   ReduceScatter: recv_r[i] = rank-ordered op over p of send_p[r*recvcount + i];
 *                  in place allowed: recvbuf == sendbuf + rank*recvcount.
 *   AllGather:     recv[p*sendcount + i] = send_p[i] on every rank;
 *                  in place allowed: sendbuf == recvbuf + rank*sendcount.
 *   Broadcast:     every rank's buf := root's buf.
 * Real comms (nlocal = 1) must pass REGISTERED buffers for the memory peers
 * access (RS: sendbuf, AG: recvbuf, BC: buf; same offsets on every rank) ->
 * else POLAR_EINVAL.  The _v forms take nlocal pointers (virtual comms). */
polar_status polar_reduce_scatter(polar_comm_t comm, const void* sendbuf, void* recvbuf, size_t recvcount,
                                  polar_dtype dtype, polar_op op, void* stream);
polar_status polar_reduce_scatter_v(polar_comm_t comm, void* const* sendbufs, void* const* recvbufs,
                                    size_t recvcount, polar_dtype dtype, polar_op op, void* stream);
polar_status polar_all_gather(polar_comm_t comm, const void* sendbuf, void* recvbuf, size_t sendcount,
                              polar_dtype dtype, void* stream);
polar_status polar_all_gather_v(polar_comm_t comm, void* const* sendbufs, void* const* recvbufs, size_t sendcount,
                                polar_dtype dtype, void* stream);
polar_status polar_broadcast(polar_comm_t comm, void* buf, size_t count, polar_dtype dtype, int root, void* stream);
polar_status polar_broadcast_v(polar_comm_t comm, void* const* bufs, size_t count, polar_dtype dtype, int root,
                               void* stream);

/* ----------------------------------------------------------- NVLS
 * POLAR_ALGO_NVLS reduces inside the NVSwitch (NCCL's
 * default, 836.3 GB/s at 8 GiB on the paper's node): polar_comm_init creates one
 * multicast object over the comm's GPUs (cuMulticastCreate; FABRIC handle, else
 * a POSIX fd copied with pidfd_getfd), binds POLAR_NVLS_BYTES (default 256 MiB,
 * POLAR_NVLS=0 disables) of every rank's memory to it, and an NVLS AllReduce
 * copies the message into that region, runs `multimem.ld_reduce` + `multimem.st`
 * over each rank's shard between an entry and an exit barrier, and copies the
 * result out (chunked by the region).  The switch's f32 summation order is
 * unspecified: results are within R2's bound, not bit-equal to the rank-order
 * oracle; bf16 accumulates in f32 and rounds once; integers are exact; f32
 * min / max do not exist in the switch (POLAR_EUNSUPPORTED).  Comms without a
 * multicast object (virtual comms; nodes whose driver refuses multicast) return
 * POLAR_EUNSUPPORTED for NVLS decisions.
 * polar_nvls_available: 1 while some comm of this process holds a multicast
 * object (polar_set_policy accepts NVLS rows only then).
 * polar_comm_nvls_info: *available = 1 if this comm holds one; `why` (may be
 * NULL) receives the object's description or the first failing driver call,
 * its CUresult name and the rank it failed on. */
int polar_nvls_available(void);
polar_status polar_comm_nvls_info(polar_comm_t comm, int* available, char* why, size_t len);

/* Decision used by the most recent AllReduce on this comm. */
polar_status polar_comm_last_decision(polar_comm_t comm, polar_decision* out);

/* Channels actually launched by the most recent AllReduce (a virtual comm
 * clamps the decision to co-resident CTAs / nranks) and its grid size
 * (nchannels x nlocal).  Either pointer may be NULL. */
polar_status polar_comm_launch_info(polar_comm_t comm, uint32_t* nchannels, uint32_t* grid);

/* Transport of the most recent AllReduce on this comm: POLAR_TRANSPORT_PEER
 * (kernels exchange through peer-mapped / global memory: every real comm, and
 * virtual comms for one-shot, two-shot, LL / LL128 and unaligned buffers) or
 * POLAR_TRANSPORT_CLUSTER (virtual comms, ring / tree Simple on whole 16-B packs
 * of 16-B aligned buffers: the n ranks of a channel are the n CTAs of one
 * thread-block cluster and every hop is a distributed-shared-memory store;
 * DESIGN.md §8 "Cluster transport").  Same algorithm, schedule and reduction
 * order either way.  POLAR_CLUSTER=0 (read at polar_comm_init_virtual) keeps
 * virtual comms on the peer transport; POLAR_CLUSTER_TREE_MAX (bytes per rank,
 * default: no bound) bounds the sizes that run the cluster tree. */
enum { POLAR_TRANSPORT_PEER = 0, POLAR_TRANSPORT_CLUSTER = 1 };
polar_status polar_comm_transport(polar_comm_t comm, int* transport);

/* Number of kernels this comm has launched so far (evidence for bench.py). */
uint64_t polar_comm_launches(polar_comm_t comm);

/* Latched asynchronous errors (device timeouts: POLAR_ETIMEOUT; ranks whose
 * launches disagreed: POLAR_ESTATE); POLAR_OK if none.  Does not synchronise: an
 * error becomes visible once the kernel that raised it ended (a disagreement at
 * launch k is raised by launch k + 1). */
polar_status polar_comm_check(polar_comm_t comm);

/* Diagnostics: when dev_buf is non-NULL, every CTA of every later AllReduce on
 * this comm writes 4 %globaltimer stamps (ns) to dev_buf[4*cta + k] (kernel
 * dependent points; two-shot: start, after entry barrier, loop end, exit).
 * bytes must hold nlocal*32*4 u64.  NULL disables. */
polar_status polar_comm_set_trace(polar_comm_t comm, void* dev_buf, size_t bytes);

/* ------------------------------------------- profiler -> tuner closed loop (f3) */

/* The paper's composability case study (§5.3; Listing 1
 * L311-351) rebuilt without eBPF maps: every AllReduce kernel writes its device
 * duration (%globaltimer, CTA 0) into a host-mapped telemetry ring (the
 * "profiler"); every `period` calls the comm's controller folds the completed
 * samples of the window into a mean latency m (real comms: the max over ranks,
 * gathered through the bootstrap all-gather so every rank picks the same count)
 * and updates the channel count c used by rows flagged POLAR_ROW_ADAPTIVE_NCH
 * (R15):
 *     ref = ref[c] if known else ref[c-1];
 *     if ref known and m > contention_factor * ref:   c = c_min   (back off)
 *     else: ref[c] = m; c = min(c + 1, cap)                       (ramp)
 * A window without samples (profiler off) changes nothing: c stays at c_min. */
typedef struct {
    uint32_t enabled;           /* 1: telemetry recorded and consumed ("profiler loaded") */
    uint32_t period;            /* calls per window (>= 1)                               */
    uint32_t c_min;             /* starting / back-off channel count (>= 1)              */
    uint32_t _pad;
    double contention_factor;   /* > 1                                                   */
    double latency_scale;       /* multiplies measured latencies (contention injection,   *
                                 * SPEC.md L366-368); 1.0 in production                   */
} polar_adaptive_params;

typedef struct {
    uint32_t channels;          /* current c                              */
    uint32_t contended;         /* last window judged contended           */
    uint64_t windows;           /* windows closed                         */
    uint64_t samples;           /* telemetry samples consumed             */
    double last_mean_ns;        /* mean latency of the last closed window */
} polar_adaptive_state;

/* Configure (and reset) a comm's closed loop.  Collective for real comms (same
 * params on every rank).  Default: enabled=0, period=1000, c_min=2, factor=4, scale=1. */
polar_status polar_adaptive_config(polar_comm_t comm, const polar_adaptive_params* params);
polar_status polar_adaptive_get_state(polar_comm_t comm, polar_adaptive_state* out);

/* Change only latency_scale (contention injection) without resetting the state. */
polar_status polar_adaptive_inject(polar_comm_t comm, double latency_scale);

/* Pure host simulation of the controller rule above (no comm, no GPU): window w
 * is observed at the current c and its mean is lat[w * 33 + c] ns (a table over
 * channel counts 0..32 per window; NaN or <= 0 = no samples in that window).
 * channels_out[w] = c after window w.  Used to pin the rule against the oracle. */
polar_status polar_adaptive_simulate(const polar_adaptive_params* params, uint32_t cap, const double* lat,
                                     uint32_t nwindows, uint32_t* channels_out);

const char* polar_status_string(polar_status s);

/* Library build tag, e.g. "polar 0.1 sm_100a". */
/* Hardware probe of the LL128 premise: `pairs` writer /
 * reader warp pairs on `cuda_device` stream `iters` LL128 line groups each
 * through an 8-group FIFO (writer: the product's st_ll128 after an optional
 * random delay < jitter_ns, drawn per lane (jitter_mode 0, the product's fault
 * injection), once per warp (jitter_mode 1) or as a per-lane divergent busy
 * wait without NANOSLEEP (jitter_mode 2); reader: the product's poll
 * pattern) and count reader
 * lanes whose payload does not match the sequence number the line flags
 * announced.  *torn_lanes == 0 is the premise; *lane_reads = lanes checked.
 * Synchronous; allocates and frees its own device memory.  Diagnostic only. */
polar_status polar_probe_ll128(int cuda_device, int pairs, unsigned long long iters, unsigned jitter_ns,
                               int jitter_mode, unsigned long long* torn_lanes, unsigned long long* lane_reads);

/* The same LL128 premise over a comm's OWN transport (collective; VERDICT r01
 * #6): rank r's 64 writer warps stream `iters` LL128 line groups each into rank
 * (r+1)'s scratch through the peer mapping (CUDA IPC / NVLink), rank (r+1)'s
 * reader warps poll them in place and return credits through the peer mapping.
 * *torn_lanes / *lane_reads are summed over every rank.  A real comm accepts
 * LL128 decisions (policy or forced) only after a probe found 0 torn lanes in
 * all n x 64 x iters x 32 lane reads (or with POLAR_LL128_REAL=1); until then
 * they return POLAR_EUNSUPPORTED.  Virtual comms run polar_probe_ll128 on their
 * device instead.  Synchronous; every wait bounded (POLAR_ETIMEOUT). */
polar_status polar_comm_probe_ll128(polar_comm_t comm, unsigned long long iters, unsigned long long* torn_lanes,
                                   unsigned long long* lane_reads);

/* p2p probe (§8(d) "measure it with p2p_probe, no number
 * is assumed"): the empirical peer-path roofline.  COLLECTIVE over the comm.
 * bufs: nlocal device pointers to symmetric buffers of >= bytes (polar_mem_alloc
 * on real comms, any 16-B aligned buffers on virtual comms); bytes a multiple
 * of 16.  Every rank r, all at once, (1) reads the buffer of peer (r + 1) mod n
 * `iters` times with 16-B loads through the peer mapping (NVLink/NVSwitch on a
 * real node, local HBM for virtual ranks), (2) overwrites that peer buffer
 * `iters` times with a known pattern (pack i = {i, hi32(i) ^ 0x9E3779B9, r, ~i}),
 * (3) bounces a flag `iters` times with rank r ^ 1.  Times are device
 * timestamps between an entry and an exit barrier.  out[nlocal]: per local
 * rank, load / store GB/s (bytes * iters / duration), flag round trip in us (0
 * for an unpaired last rank), and the XOR of the peer's 16-B packs as read
 * (each pack folded to 64 bits as (w0 ^ w2) << 32 | (w1 ^ w3)).  The peer
 * buffer holds the store pattern afterwards.  Synchronous.  EINVAL for bad
 * arguments or an unregistered buffer on a real comm. */
typedef struct {
    double load_gbs, store_gbs, pingpong_us;
    unsigned long long load_xor;
} polar_p2p_result;
polar_status polar_p2p_probe(polar_comm_t comm, void* const* bufs, size_t bytes, int iters, polar_p2p_result* out);

const char* polar_version(void);

#ifdef __cplusplus
}
#endif
#endif /* POLAR_H */
