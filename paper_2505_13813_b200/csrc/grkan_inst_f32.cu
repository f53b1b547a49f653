// Kernel instantiations and launchers for f32 I/O (one TU per dtype so nvcc builds them in parallel).
#include "grkan_launch.cuh"

GRKAN_DEFINE_LAUNCHERS(float, f32)
GRKAN_PROBE_EXPORTS(f32)
