// Kernel instantiation tables, one translation unit per dtype (inst_<dt>.cu;
// separate TUs so nvcc compiles the 36 kernels of each dtype in parallel).
// POLAR_INSTANTIATE(name, DT) defines kernel_<name>(op, algo, proto) and
// direct_kernel_<name>(mode, op) declared in dispatch.h.
#pragma once
#include "dispatch.h"
#include "kernels.cuh"

namespace polar {
namespace inst {

template <int DT, int OP, int ALGO, int PROTO>
const void* k() { return reinterpret_cast<const void*>(&dev::allreduce_kernel<DT, OP, ALGO, PROTO>); }

template <int DT, int OP, int PROTO>
const void* by_algo_p(int algo) {
    switch (algo) {
        case POLAR_ALGO_TWOSHOT: return k<DT, OP, POLAR_ALGO_TWOSHOT, PROTO>();
        case POLAR_ALGO_ONESHOT: return k<DT, OP, POLAR_ALGO_ONESHOT, PROTO>();
        case POLAR_ALGO_RING: return k<DT, OP, POLAR_ALGO_RING, PROTO>();
        case POLAR_ALGO_TREE: return k<DT, OP, POLAR_ALGO_TREE, PROTO>();
    }
    return nullptr;
}

template <int DT, int OP>
const void* by_algo(int algo, int proto) {
    switch (proto) {
        case POLAR_PROTO_LL: return by_algo_p<DT, OP, POLAR_PROTO_LL>(algo);
        case POLAR_PROTO_LL128: return by_algo_p<DT, OP, POLAR_PROTO_LL128>(algo);
        case POLAR_PROTO_SIMPLE: return by_algo_p<DT, OP, POLAR_PROTO_SIMPLE>(algo);
    }
    return nullptr;
}

template <int DT>
const void* kernel(int op, int algo, int proto) {
    switch (op) {
        case POLAR_SUM: return by_algo<DT, POLAR_SUM>(algo, proto);
        case POLAR_MAX: return by_algo<DT, POLAR_MAX>(algo, proto);
        case POLAR_MIN: return by_algo<DT, POLAR_MIN>(algo, proto);
    }
    return nullptr;
}

template <int DT, int OP, int MODE>
const void* d() { return reinterpret_cast<const void*>(&dev::direct_kernel<DT, OP, MODE>); }

template <int DT>
const void* direct(int mode, int op) {
    switch (mode) {
        case dev::MODE_RS:
            if (op == POLAR_SUM) return d<DT, POLAR_SUM, dev::MODE_RS>();
            if (op == POLAR_MAX) return d<DT, POLAR_MAX, dev::MODE_RS>();
            if (op == POLAR_MIN) return d<DT, POLAR_MIN, dev::MODE_RS>();
            return nullptr;
        case dev::MODE_AG: return d<DT, POLAR_SUM, dev::MODE_AG>();
        case dev::MODE_BC: return d<DT, POLAR_SUM, dev::MODE_BC>();
    }
    return nullptr;
}

}  // namespace inst
}  // namespace polar

#define POLAR_INSTANTIATE(name, DT)                                                                     \
    namespace polar {                                                                                   \
    const void* kernel_##name(int op, int algo, int proto) { return inst::kernel<DT>(op, algo, proto); } \
    const void* direct_kernel_##name(int mode, int op) { return inst::direct<DT>(mode, op); }            \
    }
