// NVLS: AllReduce reduced inside the NVSwitch (the algorithm
// NCCL picks by default on the paper's B300 node and the best one from 256 MiB
// on: 836.3 GB/s = 92.9 % of 900 at 8 GiB, Table 2).
//
// Every rank's copy of the message lives in memory bound to ONE multicast object
// (nvls_host.cpp).  Rank r owns shard r of the packs; for each 16-B pack of its
// shard one `multimem.ld_reduce` through the multicast address makes the switch
// read that pack from every rank and return the reduction, and one `multimem.st`
// makes the switch write the result into every rank's copy.  Per rank on NVLink:
// (n-1)/n S in + (n-1)/n S out — the reduction happens in the switch, so busBW
// can exceed the 2(n-1)/n S ring / two-shot bound (NCCL's NVLS figure).
//
// Between an entry barrier (every rank's input is in its bound copy; the
// barrier also exchanges the decision tag, kernels.cuh handshake_entry) and an
// exit barrier (every store of every rank performed).  Inputs are written and
// results read through the UNICAST mapping of the same physical memory:
// `fence.proxy.alias` orders those accesses with the multicast ones.
//
// Precision: the switch's reduction order is unspecified, so f32 sums are held
// to R2's bound (1e-6 n sum|x|), not to bit equality; bf16 accumulates in f32
// (`.acc::f32`) with one rounding; integers wrap and are exact.  The switch has
// no f32 min / max: those combinations do not exist (nvls_kernel_for -> null ->
// POLAR_EUNSUPPORTED).
#include "dispatch.h"
#include "kernels.cuh"

namespace polar {
namespace dev {

__device__ __forceinline__ void fence_proxy_alias() { asm volatile("fence.proxy.alias;" ::: "memory"); }

// one 16-B pack: reduce it across every rank's bound copy, then store the result to all
template <int DT, int OP>
__device__ __forceinline__ uint4 mm_ld_reduce(const char* mc) {
    uint4 v;
    if constexpr (DT == POLAR_FLOAT32) {
        static_assert(OP == POLAR_SUM, "the switch reduces f32 by add only");
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(mc) : "memory");
    } else if constexpr (DT == POLAR_BFLOAT16) {
        if constexpr (OP == POLAR_SUM)
            asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(mc) : "memory");
        else if constexpr (OP == POLAR_MAX)
            asm volatile("multimem.ld_reduce.relaxed.sys.global.max.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(mc) : "memory");
        else
            asm volatile("multimem.ld_reduce.relaxed.sys.global.min.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(mc) : "memory");
    } else if constexpr (DT == POLAR_INT32) {
        uint32_t* o = &v.x;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if constexpr (OP == POLAR_SUM)
                asm volatile("multimem.ld_reduce.relaxed.sys.global.add.u32 %0, [%1];" : "=r"(o[k]) : "l"(mc + 4 * k) : "memory");
            else if constexpr (OP == POLAR_MAX)
                asm volatile("multimem.ld_reduce.relaxed.sys.global.max.s32 %0, [%1];" : "=r"(o[k]) : "l"(mc + 4 * k) : "memory");
            else
                asm volatile("multimem.ld_reduce.relaxed.sys.global.min.s32 %0, [%1];" : "=r"(o[k]) : "l"(mc + 4 * k) : "memory");
        }
    } else {
        unsigned long long a[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            if constexpr (OP == POLAR_SUM)
                asm volatile("multimem.ld_reduce.relaxed.sys.global.add.u64 %0, [%1];" : "=l"(a[k]) : "l"(mc + 8 * k) : "memory");
            else if constexpr (OP == POLAR_MAX)
                asm volatile("multimem.ld_reduce.relaxed.sys.global.max.s64 %0, [%1];" : "=l"(a[k]) : "l"(mc + 8 * k) : "memory");
            else
                asm volatile("multimem.ld_reduce.relaxed.sys.global.min.s64 %0, [%1];" : "=l"(a[k]) : "l"(mc + 8 * k) : "memory");
        }
        v = make_uint4((uint32_t)a[0], (uint32_t)(a[0] >> 32), (uint32_t)a[1], (uint32_t)(a[1] >> 32));
    }
    return v;
}
__device__ __forceinline__ void mm_st(char* mc, uint4 v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

// P.bufs[rank0] = this rank's bound copy (unicast), P.recv[0] = the same offset
// through the multicast mapping; P.count elements; whole 16-B packs (the bound
// region is padded, so a partial last pack reduces padding that is never copied out).
template <int DT, int OP>
__global__ void __launch_bounds__(kBlock, POLAR_LB_MIN) nvls_kernel(Params P) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    constexpr int ES = DType<DT>::ES;
    __shared__ __align__(16) uint4 s_tags[kMaxRanks];
    tag_begin(P, s_tags);
    const Who w = who(P);
    ChanState* st = chan_state(P, w.r, w.c);
    const uint64_t e = st->epoch + 1;
    fence_proxy_alias();                 // inputs written through the unicast mapping
    if (!handshake_entry(P, w, e)) return;
    unsigned long long s0, s1, a, b;
    split_range(0, npacks<ES>(P), w.n, w.r, s0, s1);
    split_range(s0, s1, P.nch, w.c, a, b);
    char* mc = P.recv[0];
    constexpr int U = 4;                 // loads in flight per thread
    const unsigned long long stride = blockDim.x;
    for (unsigned long long i0 = a + threadIdx.x; i0 < b; i0 += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + u * stride < b) v[u] = mm_ld_reduce<DT, OP>(mc + (i0 + u * stride) * 16);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + u * stride < b) mm_st(mc + (i0 + u * stride) * 16, v[u]);
    }
    __syncthreads();
    if (!handshake_exit(P, w, e)) return;   // every rank's multimem stores are performed
    fence_proxy_alias();                     // results read back through the unicast mapping
    epoch_publish(P, w, e);
    tag_end(P, s_tags);
}

}  // namespace dev

template <int DT>
static const void* nvls_by_op(int op) {
    using namespace dev;
    if constexpr (DT == POLAR_FLOAT32) {
        return op == POLAR_SUM ? reinterpret_cast<const void*>(&nvls_kernel<DT, POLAR_SUM>) : nullptr;
    } else {
        switch (op) {
            case POLAR_SUM: return reinterpret_cast<const void*>(&nvls_kernel<DT, POLAR_SUM>);
            case POLAR_MAX: return reinterpret_cast<const void*>(&nvls_kernel<DT, POLAR_MAX>);
            case POLAR_MIN: return reinterpret_cast<const void*>(&nvls_kernel<DT, POLAR_MIN>);
        }
        return nullptr;
    }
}

const void* nvls_kernel_for(int dtype, int op) {
    switch (dtype) {
        case POLAR_INT32: return nvls_by_op<POLAR_INT32>(op);
        case POLAR_INT64: return nvls_by_op<POLAR_INT64>(op);
        case POLAR_FLOAT32: return nvls_by_op<POLAR_FLOAT32>(op);
        case POLAR_BFLOAT16: return nvls_by_op<POLAR_BFLOAT16>(op);
    }
    return nullptr;
}

}  // namespace polar
