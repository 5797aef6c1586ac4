// Kernel table: one instantiation per <dtype, op, algorithm, protocol>, compiled
// in inst_<dtype>.cu (one translation unit per dtype so nvcc runs in parallel).
#pragma once
#include <cstddef>

#include "polar.h"

namespace polar {

// nullptr if the combination does not exist
const void* kernel_i32(int op, int algo, int proto);
const void* kernel_i64(int op, int algo, int proto);
const void* kernel_f32(int op, int algo, int proto);
const void* kernel_bf16(int op, int algo, int proto);
const void* init_barrier_kernel_ptr();
// direct collectives: mode 0 = ReduceScatter (op used), 1 = AllGather, 2 = Broadcast
const void* direct_kernel_i32(int mode, int op);
const void* direct_kernel_i64(int mode, int op);
const void* direct_kernel_f32(int mode, int op);
const void* direct_kernel_bf16(int mode, int op);

// NVLS (switch reduction, nvls.cu): nullptr where the switch has no such
// reduction (f32 min / max)
const void* nvls_kernel_for(int dtype, int op);

// Cluster-transport ring / tree Simple for virtual comms (cluster.cu): nullptr
// where no cluster kernel exists; its dynamic shared memory and block size
const void* cluster_kernel_for(int dtype, int op, int algo);
size_t cluster_smem_bytes(int algo);
int cluster_threads(int algo);

inline const void* direct_kernel_for(int dtype, int mode, int op) {
    switch (dtype) {
        case POLAR_INT32: return direct_kernel_i32(mode, op);
        case POLAR_INT64: return direct_kernel_i64(mode, op);
        case POLAR_FLOAT32: return direct_kernel_f32(mode, op);
        case POLAR_BFLOAT16: return direct_kernel_bf16(mode, op);
    }
    return nullptr;
}

inline const void* kernel_for(int dtype, int op, int algo, int proto) {
    switch (dtype) {
        case POLAR_INT32: return kernel_i32(op, algo, proto);
        case POLAR_INT64: return kernel_i64(op, algo, proto);
        case POLAR_FLOAT32: return kernel_f32(op, algo, proto);
        case POLAR_BFLOAT16: return kernel_bf16(op, algo, proto);
    }
    return nullptr;
}

}  // namespace polar
