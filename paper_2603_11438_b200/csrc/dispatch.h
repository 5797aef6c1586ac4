// Kernel table: one instantiation per <dtype, op, algorithm, protocol>, compiled
// in inst_<dtype>.cu (one translation unit per dtype so nvcc runs in parallel).
#pragma once
#include "polar.h"

namespace polar {

// nullptr if the combination does not exist
const void* kernel_i32(int op, int algo, int proto);
const void* kernel_i64(int op, int algo, int proto);
const void* kernel_f32(int op, int algo, int proto);
const void* kernel_bf16(int op, int algo, int proto);
const void* init_barrier_kernel_ptr();

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
