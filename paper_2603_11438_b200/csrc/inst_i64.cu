// Kernel instantiations for dtype POLAR_INT64 (inst.cuh, dispatch.h).
#include "inst.cuh"

POLAR_INSTANTIATE(i64, POLAR_INT64)
