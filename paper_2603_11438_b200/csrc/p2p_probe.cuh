// p2p probe (SURVEY.md §2.4 K7, §8(d) "Measure it with p2p_probe ping-pong; no
// number is assumed here"): the empirical roofline of the peer path the
// AllReduce kernels use — 16-B loads from and stores to a peer's symmetric
// buffer through the same peer mapping (NVLink/NVSwitch on a real node, local
// HBM for virtual ranks), and the flag round-trip latency between two ranks.
// Every rank r pairs with peer (r + 1) mod n for load/store (all ranks at once:
// the per-GPU egress/ingress pattern of ring and two-shot) and with r ^ 1 for
// the ping-pong.  Diagnostic / measurement kernel; not on the AllReduce path.
#pragma once
#include "device.cuh"

namespace polar {
namespace dev {

enum { PROBE_LOAD = 0, PROBE_STORE = 1, PROBE_PINGPONG = 2 };

// the pattern rank `writer` stores at pack i of its peer's buffer
__device__ __forceinline__ uint4 probe_pattern(unsigned long long i, int writer) {
    return make_uint4((uint32_t)i, (uint32_t)(i >> 32) ^ 0x9E3779B9u, (uint32_t)writer, ~(uint32_t)i);
}

// times[2 b] / times[2 b + 1]: %globaltimer after the entry barrier / before the
// exit barrier of CTA b; sums[b]: XOR of every pack loaded (load mode)
__global__ void __launch_bounds__(kBlock, 1)
p2p_probe_kernel(Params P, int mode, int iters, unsigned long long epoch, unsigned long long* times,
                 unsigned long long* sums) {
    const int r = P.rank0 + (int)blockIdx.x / P.nch, c = (int)blockIdx.x % P.nch;
    const int n = P.nranks, tid = (int)threadIdx.x;
    if (tid < n) st_release(flag_ptr(P, tid, F_PROBE_ENTRY, c, r), epoch, P.sys);
    bool ok = true;
    if (tid < n) ok = wait_geq(P, flag_ptr(P, r, F_PROBE_ENTRY, c, tid), epoch);
    if (!__syncthreads_and(ok)) return;
    unsigned long long t0 = globaltimer();
    const int peer = (r + 1) % n;
    const unsigned long long NP = P.count / 16;
    unsigned long long a, b;
    split_range(0, NP, P.nch, c, a, b);
    const unsigned long long B = blockDim.x;
    if (mode == PROBE_LOAD) {
        const uint4* src = reinterpret_cast<const uint4*>(P.bufs[peer]);
        uint4 x = make_uint4(0, 0, 0, 0);
        for (int it = 0; it < iters; ++it) {
            x = make_uint4(0, 0, 0, 0);   // keep the last pass's XOR (every pass loads every pack)
            for (unsigned long long i0 = a + tid; i0 < b; i0 += 4 * B) {
                uint4 v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (i0 + u * B < b) v[u] = ld_cg(src + i0 + u * B);
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (i0 + u * B < b) { x.x ^= v[u].x; x.y ^= v[u].y; x.z ^= v[u].z; x.w ^= v[u].w; }
            }
        }
        // CTA-wide XOR of the packs of the last pass
        unsigned long long w = ((unsigned long long)(x.x ^ x.z) << 32) | (x.y ^ x.w);
        for (int o = 16; o; o >>= 1) w ^= __shfl_xor_sync(0xffffffffu, w, o);
        __shared__ unsigned long long red[kBlock / 32];
        if ((tid & 31) == 0) red[tid >> 5] = w;
        __syncthreads();
        if (tid == 0) {
            unsigned long long t = 0;
            for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t ^= red[k];
            sums[blockIdx.x] = t;
        }
    } else if (mode == PROBE_STORE) {
        uint4* dst = reinterpret_cast<uint4*>(P.bufs[peer]);
        for (int it = 0; it < iters; ++it)
            for (unsigned long long i = a + tid; i < b; i += B) st_plain(dst + i, probe_pattern(i, r));
    } else if (c == 0 && tid == 0 && (r ^ 1) < n) {
        const int q = r ^ 1;
        uint64_t* mine = flag_ptr(P, r, F_PROBE_PP, 0, 0);
        uint64_t* theirs = flag_ptr(P, q, F_PROBE_PP, 0, 0);
        const unsigned long long base = epoch * (unsigned long long)(iters + 1);
        for (int k = 1; k <= iters && ok; ++k) {
            if ((r & 1) == 0) {
                st_relaxed(theirs, base + k, P.sys);
                ok = wait_geq(P, mine, base + k);
            } else {
                ok = wait_geq(P, mine, base + k);
                if (ok) st_relaxed(theirs, base + k, P.sys);
            }
        }
    }
    __syncthreads();
    unsigned long long t1 = globaltimer();
    if (tid == 0) {
        times[2 * blockIdx.x] = t0;
        times[2 * blockIdx.x + 1] = t1;
    }
    if (tid < n) {
        fence_acq_rel(P.sys);
        st_relaxed(flag_ptr(P, tid, F_PROBE_EXIT, c, r), epoch, P.sys);
    }
    ok = true;
    if (tid < n) ok = wait_geq(P, flag_ptr(P, r, F_PROBE_EXIT, c, tid), epoch);
    __syncthreads_and(ok);
}

}  // namespace dev
}  // namespace polar
