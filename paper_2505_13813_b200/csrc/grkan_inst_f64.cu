// Kernel instantiations and launchers for f64 I/O (one TU per dtype so nvcc builds them in parallel).
#include "grkan_launch.cuh"

GRKAN_DEFINE_LAUNCHERS(double, f64)
GRKAN_PROBE_EXPORTS(f64)
