// Kernel instantiations for dtype POLAR_FLOAT32 (see dispatch.h).
#include "dispatch.h"
#include "kernels.cuh"

namespace polar {

template <int OP, int ALGO, int PROTO>
static const void* k() { return reinterpret_cast<const void*>(&dev::allreduce_kernel<POLAR_FLOAT32, OP, ALGO, PROTO>); }

template <int OP, int PROTO>
static const void* by_algo_p(int algo) {
    switch (algo) {
        case POLAR_ALGO_TWOSHOT: return k<OP, POLAR_ALGO_TWOSHOT, PROTO>();
        case POLAR_ALGO_ONESHOT: return k<OP, POLAR_ALGO_ONESHOT, PROTO>();
        case POLAR_ALGO_RING: return k<OP, POLAR_ALGO_RING, PROTO>();
        case POLAR_ALGO_TREE: return k<OP, POLAR_ALGO_TREE, PROTO>();
    }
    return nullptr;
}

template <int OP>
static const void* by_algo(int algo, int proto) {
    switch (proto) {
        case POLAR_PROTO_LL: return by_algo_p<OP, POLAR_PROTO_LL>(algo);
        case POLAR_PROTO_LL128: return by_algo_p<OP, POLAR_PROTO_LL128>(algo);
        case POLAR_PROTO_SIMPLE: return by_algo_p<OP, POLAR_PROTO_SIMPLE>(algo);
    }
    return nullptr;
}

const void* kernel_f32(int op, int algo, int proto) {
    switch (op) {
        case POLAR_SUM: return by_algo<POLAR_SUM>(algo, proto);
        case POLAR_MAX: return by_algo<POLAR_MAX>(algo, proto);
        case POLAR_MIN: return by_algo<POLAR_MIN>(algo, proto);
    }
    return nullptr;
}

const void* direct_kernel_f32(int mode, int op) {
    using namespace dev;
    switch (mode) {
        case MODE_RS:
            if (op == POLAR_SUM) return reinterpret_cast<const void*>(&direct_kernel<POLAR_FLOAT32, POLAR_SUM, MODE_RS>);
            if (op == POLAR_MAX) return reinterpret_cast<const void*>(&direct_kernel<POLAR_FLOAT32, POLAR_MAX, MODE_RS>);
            if (op == POLAR_MIN) return reinterpret_cast<const void*>(&direct_kernel<POLAR_FLOAT32, POLAR_MIN, MODE_RS>);
            return nullptr;
        case MODE_AG: return reinterpret_cast<const void*>(&direct_kernel<POLAR_FLOAT32, POLAR_SUM, MODE_AG>);
        case MODE_BC: return reinterpret_cast<const void*>(&direct_kernel<POLAR_FLOAT32, POLAR_SUM, MODE_BC>);
    }
    return nullptr;
}

}  // namespace polar
