// Kernel instantiations for dtype POLAR_FLOAT32 (inst.cuh, dispatch.h).
#include "inst.cuh"

POLAR_INSTANTIATE(f32, POLAR_FLOAT32)
