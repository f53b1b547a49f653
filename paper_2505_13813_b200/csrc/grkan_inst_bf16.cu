// Kernel instantiations and launchers for bf16 I/O (one TU per dtype so nvcc builds them in parallel).
#include "grkan_launch.cuh"

GRKAN_DEFINE_LAUNCHERS(__nv_bfloat16, bf16)
GRKAN_PROBE_EXPORTS(bf16)
