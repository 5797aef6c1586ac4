// Kernel instantiations for dtype POLAR_INT32 (inst.cuh, dispatch.h).
#include "inst.cuh"

POLAR_INSTANTIATE(i32, POLAR_INT32)
