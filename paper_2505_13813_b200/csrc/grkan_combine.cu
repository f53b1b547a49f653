// grkan_combine.cu -- the reference's combine_partials fold, bit for bit, on the device.
//
// combine_partials (pkg/src/grkan/backward.py:142-179) folds per-block partials into
// per-group totals with `d_a[g] += pa` from zeros, in ascending block_id order
// (deterministic_ordered) or in the order given (unordered_scatter), IN THE PARTIALS'
// DTYPE -- so its rounding, including absorption of tiny partials into a large
// running total (pkg/tests/test_backward.py:193-209), is part of the contract.  K3
// (k_bwd_reduce) folds in fp64 with a tree, which is more accurate but not that
// result; this kernel is the contract itself: one thread per (group, coefficient)
// walks the entries in fold order with separately rounded adds in the dtype.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>

#include "../../include/grkan_b200.h"
#include "grkan_types.h"

namespace {

template <typename A>
__device__ __forceinline__ A add_rn(A a, A b);
template <>
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

// part[i * kc + k] for entry i in fold order; group_of[i] = block_id % n_groups.
template <typename A>
__global__ void k_combine_ordered(const A* __restrict__ part, const int32_t* __restrict__ group_of, int64_t n,
                                  int ng, int num_w, int den_w, A* __restrict__ da, A* __restrict__ db) {
  const int kc = num_w + den_w;
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= ng * kc) return;
  const int g = col / kc, k = col % kc;
  A s = A(0);
  for (int64_t i = 0; i < n; ++i)
    if (group_of[i] == g) s = add_rn(s, part[i * kc + k]);
  if (k < num_w)
    da[g * num_w + k] = s;
  else
    db[g * den_w + (k - num_w)] = s;
}

int cfail(int code, const char* fmt, ...) {
  char buf[256];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return grkan::set_error(code, buf);
}

}  // namespace

extern "C" {

int grkan_combine_partials(const void* part, const int32_t* group_of, int64_t n_entries, int32_t n_groups,
                           int32_t num_w, int32_t den_w, void* da, void* db, int32_t dtype, void* stream) {
  if (n_groups < 1 || num_w < 0 || den_w < 0 || n_entries < 0)
    return cfail(GRKAN_ERR_INVALID, "invalid combine geometry");
  if (dtype != GRKAN_F32 && dtype != GRKAN_F64)
    return cfail(GRKAN_ERR_UNSUPPORTED, "combine_partials folds float32 or float64 partials");
  const int cols = n_groups * (num_w + den_w);
  if (cols == 0) return GRKAN_OK;
  if ((n_entries > 0 && (!part || !group_of)) || (num_w > 0 && !da) || (den_w > 0 && !db))
    return cfail(GRKAN_ERR_INVALID, "null pointer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const unsigned blocks = static_cast<unsigned>((cols + 127) / 128);
  if (dtype == GRKAN_F32)
    k_combine_ordered<float><<<blocks, 128, 0, s>>>(static_cast<const float*>(part), group_of, n_entries, n_groups,
                                                    num_w, den_w, static_cast<float*>(da), static_cast<float*>(db));
  else
    k_combine_ordered<double><<<blocks, 128, 0, s>>>(static_cast<const double*>(part), group_of, n_entries,
                                                     n_groups, num_w, den_w, static_cast<double*>(da),
                                                     static_cast<double*>(db));
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cfail(GRKAN_ERR_CUDA, "k_combine_ordered: %s", cudaGetErrorString(e));
  return GRKAN_OK;
}

}  // extern "C"
