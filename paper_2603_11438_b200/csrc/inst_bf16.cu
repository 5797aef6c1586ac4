// Kernel instantiations for dtype POLAR_BFLOAT16 (inst.cuh, dispatch.h).
#include "inst.cuh"

POLAR_INSTANTIATE(bf16, POLAR_BFLOAT16)
