// Hardware probe for the LL128 premise: does a reader that
// sees a line's flag also see the rest of that 128-B line?  Writer warps stream
// sequence-numbered line groups (st_ll128, the product's store) into a FIFO of
// K groups; reader warps poll each group with the product's load pattern and
// count lanes whose payload does not belong to the sequence number the flags
// announced ("torn" reads).  Diagnostic entry point, not on the hot path.
#include <cuda_runtime.h>

#include "device.cuh"
#include "polar.h"

namespace polar {
namespace dev {

constexpr int kProbeSlots = 8;   // line groups per writer/reader pair

__global__ void probe_ll128_kernel(uint4* fifo, unsigned long long* credits, unsigned long long iters,
                                   unsigned jitter_ns, int mode, unsigned long long* torn, unsigned long long* reads) {
    // blocks come in pairs: 2p writes, 2p+1 reads; one warp each
    const int pair = blockIdx.x >> 1;
    const bool writer = (blockIdx.x & 1) == 0;
    const int lane = threadIdx.x & 31, q = lane & 7;
    uint4* base = fifo + (size_t)pair * kProbeSlots * 32;
    unsigned long long* credit = credits + (size_t)pair * 16;
    Params P;
    memset(&P, 0, sizeof(P));
    P.jitter_ns = jitter_ns;
    unsigned long long bad = 0, nread = 0;
    for (unsigned long long s = 1; s <= iters; ++s) {
        uint4* g = base + (s % kProbeSlots) * 32;
        if (writer) {
            if (s > kProbeSlots) {
                // wait until the reader consumed sequence s - K (slot reuse)
                while (true) {
                    unsigned long long c;
                    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(c) : "l"(credit) : "memory");
                    if (__all_sync(0xffffffffu, c >= s - kProbeSlots)) break;
                }
            }
            // lane L < 30 holds pack L = 4 copies of s*131 + L (the unit's packing)
            const uint32_t pk = (uint32_t)(s * 131u + (unsigned)(lane < 30 ? lane : 0));
            if (mode == 0) {
                jitter(P);   // per-lane random delay (NANOSLEEP, the LL/Simple fault injection)
            } else if (mode == 2 && jitter_ns) {
                // per-lane divergent busy wait (no NANOSLEEP): data-dependent divergence
                uint32_t x = (uint32_t)globaltimer() * 2654435761u ^ ((unsigned)lane * 40503u) ^ (blockIdx.x * 2246822519u);
                x ^= x >> 15; x *= 2246822519u; x ^= x >> 13;
                if ((x & 7u) == 0) {
                    const uint64_t t0 = globaltimer();
                    while (globaltimer() - t0 < x % jitter_ns) {}
                }
            } else if (jitter_ns) {
                // warp-uniform delay: lane 0 draws, every lane sleeps the same time
                uint32_t x = (uint32_t)globaltimer() * 2654435761u ^ (blockIdx.x * 2246822519u);
                x ^= x >> 15; x *= 2246822519u; x ^= x >> 13;
                x = __shfl_sync(0xffffffffu, x, 0);
                if ((x & 7u) == 0) __nanosleep(x % jitter_ns);
            }
            __syncwarp();
            st_ll128(g, make_uint4(pk, pk, pk, pk), s);
        } else {
            uint4 w;
            const uint32_t flo = (uint32_t)s, fhi = (uint32_t)(s >> 32);
            while (true) {
                w = ld_ll(g + lane);
                const bool mine = q != 7 || (w.z == flo && w.w == fhi);
                if (__all_sync(0xffffffffu, mine)) break;
            }
            // which pack does lane hold in the line layout: q < 7 -> pack 7g+q (4 words),
            // q == 7 -> half of pack 28 + g/2 (2 words)
            const int gi = lane >> 3;
            const uint32_t pk = (uint32_t)(s * 131u + (unsigned)(q < 7 ? gi * 7 + q : 28 + (gi >> 1)));
            bool ok = w.x == pk && w.y == pk;
            if (q < 7) ok = ok && w.z == pk && w.w == pk;
            bad += ok ? 0 : 1;
            nread += 1;
            __syncwarp();
            if (lane == 0) asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(credit), "l"(s) : "memory");
        }
    }
    if (!writer) {
        atomicAdd(torn, bad);
        atomicAdd(reads, nread);
    }
}

}  // namespace dev
}  // namespace polar

extern "C" polar_status polar_probe_ll128(int cuda_device, int pairs, unsigned long long iters, unsigned jitter_ns,
                                          int jitter_mode, unsigned long long* torn_lanes,
                                          unsigned long long* lane_reads) {
    if (pairs < 1 || pairs > 1024 || !torn_lanes || !lane_reads) return POLAR_EINVAL;
    int prev = -1;
    cudaGetDevice(&prev);
    if (cudaSetDevice(cuda_device) != cudaSuccess) return POLAR_ECUDA;
    polar_status st = POLAR_OK;
    uint4* fifo = nullptr;
    unsigned long long *credits = nullptr, *cnt = nullptr;
    const size_t fifo_bytes = (size_t)pairs * polar::dev::kProbeSlots * 512;
    if (cudaMalloc(&fifo, fifo_bytes) != cudaSuccess || cudaMalloc(&credits, (size_t)pairs * 128) != cudaSuccess ||
        cudaMalloc(&cnt, 16) != cudaSuccess) {
        st = POLAR_ENOMEM;
    } else {
        cudaMemset(fifo, 0, fifo_bytes);
        cudaMemset(credits, 0, (size_t)pairs * 128);
        cudaMemset(cnt, 0, 16);
        void* args[] = {&fifo, &credits, &iters, &jitter_ns, nullptr, &cnt, nullptr};
        int mode = jitter_mode;
        unsigned long long* reads = cnt + 1;
        args[4] = &mode;
        args[6] = &reads;
        // cooperative: writer and reader of a pair must be co-resident
        if (cudaLaunchCooperativeKernel((const void*)polar::dev::probe_ll128_kernel, dim3(2 * pairs), dim3(32), args,
                                        0, 0) != cudaSuccess ||
            cudaDeviceSynchronize() != cudaSuccess) {
            st = POLAR_ECUDA;
        } else {
            unsigned long long h[2];
            cudaMemcpy(h, cnt, 16, cudaMemcpyDeviceToHost);
            *torn_lanes = h[0];
            *lane_reads = h[1];
        }
    }
    if (fifo) cudaFree(fifo);
    if (credits) cudaFree(credits);
    if (cnt) cudaFree(cnt);
    if (prev >= 0) cudaSetDevice(prev);
    return st;
}

// ------------------------------------------------------------------ across ranks
// The same premise over a comm's transport: rank r's writer
// warps stream LL128 line groups into rank (r+1)'s probe FIFO through the peer
// mapping (CUDA IPC; NVLink on a node), rank (r+1)'s reader warps poll them in
// their own memory and return credits through the peer mapping.  Blocks
// [0, pairs) write to the next rank, [pairs, 2 pairs) read from the previous
// one.  Every spin is bounded (timeout latches into *err and ends the probe).
namespace polar {
namespace dev {

__global__ void probe_ll128_xrank_kernel(uint4* fifo_out, unsigned long long* credit_in, uint4* fifo_in,
                                         unsigned long long* credit_out, int pairs, unsigned long long iters,
                                         unsigned long long* cnt, unsigned long long timeout_ns, int* err) {
    const bool writer = (int)blockIdx.x < pairs;
    const int pair = writer ? (int)blockIdx.x : (int)blockIdx.x - pairs;
    const int lane = threadIdx.x & 31, q = lane & 7;
    uint4* base = (writer ? fifo_out : fifo_in) + (size_t)pair * kProbeSlots * 32;
    unsigned long long* credit = (writer ? credit_in : credit_out) + (size_t)pair * 16;
    unsigned long long bad = 0, nread = 0;
    const uint64_t t0 = globaltimer();
    bool dead = false;
    for (unsigned long long s = 1; s <= iters && !dead; ++s) {
        uint4* g = base + (s % kProbeSlots) * 32;
        if (writer) {
            if (s > kProbeSlots) {
                for (uint32_t it = 0;; ++it) {
                    unsigned long long c;
                    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(c) : "l"(credit) : "memory");
                    if (__all_sync(0xffffffffu, c >= s - kProbeSlots)) break;
                    if ((it & 1023) == 1023 && __any_sync(0xffffffffu, globaltimer() - t0 > timeout_ns || *(volatile int*)err)) {
                        dead = true;
                        break;
                    }
                }
                if (dead) break;
            }
            const uint32_t pk = (uint32_t)(s * 131u + (unsigned)(lane < 30 ? lane : 0));
            __syncwarp();
            st_ll128(g, make_uint4(pk, pk, pk, pk), s);
        } else {
            uint4 w;
            const uint32_t flo = (uint32_t)s, fhi = (uint32_t)(s >> 32);
            for (uint32_t it = 0;; ++it) {
                w = ld_ll(g + lane);
                const bool mine = q != 7 || (w.z == flo && w.w == fhi);
                if (__all_sync(0xffffffffu, mine)) break;
                if ((it & 1023) == 1023 && __any_sync(0xffffffffu, globaltimer() - t0 > timeout_ns || *(volatile int*)err)) {
                    dead = true;
                    break;
                }
            }
            if (dead) break;
            const int gi = lane >> 3;
            const uint32_t pk = (uint32_t)(s * 131u + (unsigned)(q < 7 ? gi * 7 + q : 28 + (gi >> 1)));
            bool ok = w.x == pk && w.y == pk;
            if (q < 7) ok = ok && w.z == pk && w.w == pk;
            bad += ok ? 0 : 1;
            nread += 1;
            __syncwarp();
            if (lane == 0) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(credit), "l"(s) : "memory");
        }
    }
    if (dead && lane == 0) {
        *(volatile int*)err = POLAR_ETIMEOUT;
        __threadfence_system();
    }
    if (!writer) {
        atomicAdd(cnt, bad);
        atomicAdd(cnt + 1, nread);
    }
}

}  // namespace dev

cudaError_t launch_probe_ll128_xrank(uint4* fifo_out, unsigned long long* credit_in, uint4* fifo_in,
                                     unsigned long long* credit_out, int pairs, unsigned long long iters,
                                     unsigned long long* cnt, unsigned long long timeout_ns, int* err) {
    dev::probe_ll128_xrank_kernel<<<2 * pairs, 32>>>(fifo_out, credit_in, fifo_in, credit_out, pairs, iters, cnt,
                                                     timeout_ns, err);
    return cudaGetLastError();
}

size_t probe_ll128_region_bytes(int pairs) { return (size_t)pairs * dev::kProbeSlots * 512 + (size_t)pairs * 128; }

}  // namespace polar
