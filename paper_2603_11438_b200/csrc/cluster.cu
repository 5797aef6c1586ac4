// Cluster-transport ring / tree Simple instantiations for virtual comms
// (cluster.cuh; DESIGN.md §8 "Cluster transport").
#include "cluster.cuh"
#include "dispatch.h"

namespace polar {

template <int DT, int OP>
static const void* ring_cl() { return reinterpret_cast<const void*>(&dev::ring_cluster_kernel<DT, OP>); }

template <int DT, int OP>
static const void* tree_cl() { return reinterpret_cast<const void*>(&dev::tree_cluster_kernel<DT, OP>); }

template <int DT>
static const void* by_op(int op, int algo) {
    if (algo == POLAR_ALGO_RING) {
        switch (op) {
            case POLAR_SUM: return ring_cl<DT, POLAR_SUM>();
            case POLAR_MAX: return ring_cl<DT, POLAR_MAX>();
            case POLAR_MIN: return ring_cl<DT, POLAR_MIN>();
        }
    } else if (algo == POLAR_ALGO_TREE) {
        switch (op) {
            case POLAR_SUM: return tree_cl<DT, POLAR_SUM>();
            case POLAR_MAX: return tree_cl<DT, POLAR_MAX>();
            case POLAR_MIN: return tree_cl<DT, POLAR_MIN>();
        }
    }
    return nullptr;
}

const void* cluster_kernel_for(int dtype, int op, int algo) {
    switch (dtype) {
        case POLAR_INT32: return by_op<POLAR_INT32>(op, algo);
        case POLAR_INT64: return by_op<POLAR_INT64>(op, algo);
        case POLAR_FLOAT32: return by_op<POLAR_FLOAT32>(op, algo);
        case POLAR_BFLOAT16: return by_op<POLAR_BFLOAT16>(op, algo);
    }
    return nullptr;
}

size_t cluster_smem_bytes(int algo) {
    return algo == POLAR_ALGO_RING ? dev::cl_ring_smem_bytes() : dev::cl_tree_smem_bytes();
}
int cluster_threads(int algo) { return algo == POLAR_ALGO_RING ? dev::kClThreads : dev::kTrThreads; }

}  // namespace polar
