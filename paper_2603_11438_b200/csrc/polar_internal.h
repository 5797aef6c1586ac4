// Internal declarations shared by the host C++ files of libpolar (not installed).
#pragma once
#include <cstddef>
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "polar.h"

namespace polar {

polar_status validate_rows(const polar_policy_row* rows, uint32_t nrows);
polar_status decide_rows(const polar_policy_row* rows, uint32_t nrows, uint32_t generation,
                         const polar_ctx* ctx, polar_decision* out);

// ----------------------------------------------------------- scratch layout
// Every rank's scratch has the same layout (offsets identical on all ranks), so a
// peer's region is peer_scratch[p] + offset.
constexpr int kMaxRanks = POLAR_MAXRANKS;
constexpr int kMaxCh = POLAR_MAXCH;

// flag kinds: one 128 B row (8 peers x u64, padded) per (kind, channel)
enum FlagKind : int {
    F_ENTRY = 0,     // two-shot: "my buffer is ready"           (written by peer p into slot p)
    F_EXIT = 1,      // two-shot: "done with your buffer"
    F_OS = 2,        // one-shot Simple: "my data is in your staging slot"
    F_RING_TAIL = 3, // ring: sender -> receiver, slots filled     (slot 0)
    F_RING_HEAD = 4, // ring: receiver -> sender, slots consumed   (slot 0)
    F_TREE_UTAIL = 5,  // tree up: child k -> parent, slot k (k = 0, 1)
    F_TREE_UHEAD = 6,  // tree up: parent -> child, slot 0
    F_TREE_DTAIL = 7,  // tree down: parent -> child, slot 0
    F_TREE_DHEAD = 8,  // tree down: child k -> parent, slot k
    F_INIT = 9,        // init barrier
    F_PROBE_ENTRY = 10,  // p2p probe: entry barrier (slot = source rank)
    F_PROBE_EXIT = 11,   // p2p probe: exit barrier
    F_PROBE_PP = 12,     // p2p probe: ping-pong flag (channel 0, slot 0)
    F_ENTRY_SIG = 13,    // zero-copy kernels: the decision tag of the launch behind F_ENTRY
    F_NKINDS = 14
};
constexpr size_t kFlagRow = 128;  // bytes per (kind, channel) row
constexpr size_t kFlagBytes = (size_t)F_NKINDS * kMaxCh * kFlagRow;

// per-channel persistent counters (local to the rank that owns the scratch)
struct ChanState {
    uint64_t epoch;        // one-shot / two-shot handshake epoch
    uint64_t ring_sent;    // slots sent to next (ring, Simple and LL share the count)
    uint64_t ring_recv;    // slots consumed from prev
    uint64_t tree_usent;   // up-slots sent to parent
    uint64_t tree_urecv[2];// up-slots consumed from child k
    uint64_t tree_dsent;   // down-slots sent to (each) child
    uint64_t tree_drecv;   // down-slots consumed from parent
    uint64_t work;         // two-shot dynamic chunk counter: (epoch << 32) | next chunk (channel 0 only)
    uint64_t pad[7];
};
constexpr size_t kStateBytes = sizeof(ChanState) * kMaxCh;
constexpr unsigned long long kTagRing = 64;   // launches remembered per rank for the decision check

struct Layout {
    size_t flags_off, state_off;
    size_t tags_off;                  // decision tags: [kTagRing] x 16 B (real comms, cross-rank check)
    size_t os_off, os_chunk;          // one-shot Simple staging: [2][kMaxRanks][os_chunk]
    size_t osll_off, osll_chunk;      // one-shot LL: [2][kMaxRanks][2*osll_chunk] (payload bytes per slot)
    size_t tsll_off, tsll_chunk;      // two-shot LL: RS [2][R][2*c] then AG [2][R][2*c]
    size_t ring_off, ring_slot;       // ring Simple FIFO: [kMaxCh][kSteps][ring_slot]
    size_t ringll_off, ringll_slot;   // ring LL FIFO: [kMaxCh][kSteps][2*ringll_slot]
    size_t tree_off, tree_slot;       // tree Simple: up [kMaxCh][2][kSteps][slot], down [kMaxCh][kSteps][slot]
    size_t treell_off, treell_slot;   // tree LL: same with 2x
    size_t os128_off;                 // one-shot LL128: [2][kMaxRanks][2*osll_chunk] (same wire bytes as LL)
    size_t ts128_off;                 // two-shot LL128: RS + AG, as two-shot LL
    size_t ring128_off, ring128_slot; // ring LL128 FIFO: [kMaxCh][kSteps][ring128_slot] (wire bytes)
    size_t tree128_off, tree128_slot; // tree LL128: up [kMaxCh][2][kSteps], down [kMaxCh][kSteps]
    size_t bounce_off, bounce_bytes;  // two-shot bounce for unregistered buffers (real comms)
    size_t probe_off;                 // LL128 premise probe across ranks (probe_ll128_region_bytes)
    size_t total;
    size_t nvls_bytes;                // NVLS region per rank (POLAR_NVLS_BYTES; 0 = NVLS off), not in scratch
};
#ifndef POLAR_FIFO_STEPS
#define POLAR_FIFO_STEPS 4
#endif
constexpr int kSteps = POLAR_FIFO_STEPS;  // FIFO depth (slots) per connection

Layout make_layout(bool with_bounce);

// LL128 premise over a comm's transport (probe.cu): kProbePairs writer/reader
// warp pairs; region = FIFO (pairs x 8 line groups) + credits (pairs x 128 B)
constexpr int kProbePairs = 64;
size_t probe_ll128_region_bytes(int pairs);
cudaError_t launch_probe_ll128_xrank(uint4* fifo_out, unsigned long long* credit_in, uint4* fifo_in,
                                     unsigned long long* credit_out, int pairs, unsigned long long iters,
                                     unsigned long long* cnt, unsigned long long timeout_ns, int* err);

// ------------------------------------------------------- NVLS (f1, nvls_host.cpp)
struct NvlsState {
    bool ok = false;                    // a multicast object is bound on every rank
    bool bound = false;
    int status = 0;                     // CUresult of the first failure (0 = none)
    int handle_type = 0;                // CUmemAllocationHandleType used to share the object
    int fd = -1;                        // rank 0, POSIX handle: kept open for the comm's life
    size_t bytes = 0;                   // bound region per rank
    unsigned long long mc_handle = 0;   // CUmemGenericAllocationHandle of the multicast object
    unsigned long long phys = 0;        // this rank's bound physical allocation
    char* uc = nullptr;                 // this rank's bound copy (unicast mapping)
    char* mc = nullptr;                 // the multicast mapping of the same region
    char why[192] = {};                 // what happened (the first failing call, or the object)
};
// Collective over the bootstrap all-gather (same number of all-gathers on every
// rank whatever fails).  POLAR_OK with s.ok == false when NVLS is unavailable
// (s.why says why); POLAR_ESTATE only if the all-gather itself failed.
polar_status nvls_setup(NvlsState& s, int nranks, int rank, int device, polar_allgather_fn ag, void* user,
                        size_t bytes);
void nvls_teardown(NvlsState& s, int device);
bool nvls_available();   // some comm of this process holds a multicast object

// ---------------------------------------------------- adaptive channels (f3)
struct Adaptive {
    polar_adaptive_params prm{};
    uint32_t c = 2;               // current channel count
    bool contended = false;
    uint64_t windows = 0, samples = 0;
    double last_mean = 0.0;
    double ref[POLAR_MAXCH + 1] = {};   // last non-contended window mean per channel count (0 = unknown)
    double win_sum = 0.0;         // samples of the open window
    uint64_t win_cnt = 0;
    uint64_t calls = 0;           // calls seen while enabled (window boundary every prm.period)
    uint32_t cap = POLAR_MAXCH;   // nchannels of the last adaptive row (the controller's cap)
};
void adaptive_reset(Adaptive& a, const polar_adaptive_params& p);
polar_status adaptive_validate(const polar_adaptive_params& p);
void adaptive_close_window(Adaptive& a, double mean_ns, uint32_t cap);

// telemetry ring entry written by the device (CTA 0 of each launch), host-mapped
struct TelEntry {
    unsigned long long seq;   // written last; == launch sequence number when t0/t1 are valid
    unsigned long long t0, t1;
    unsigned long long pad;
};
constexpr uint32_t kTelRing = 4096;

}  // namespace polar
