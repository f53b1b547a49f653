// grkan_terms.cu -- per-element gradient terms (the reference's gradient_terms,
// pkg/src/grkan/rational.py:227-278) and nothing reduced.
//
// Introspection / parity kernel, not the product path: one thread per element
// writes dx and the m1 + n per-element coefficient-gradient contributions
// (u x^i / Q and -u sign(A) x^(j+1) P / Q^2) to a [m1 + n][rows * d] buffer.
// In EXACT mode every term is bitwise the reference's (same Rational engine and
// operation order as K2); accumulators start at -0.0 so -0 + t == t keeps the
// sign of zero terms.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/grkan_b200.h"
#include "grkan_kernels.cuh"
#include "grkan_types.h"

namespace grkan {

int set_error(int code, const char* msg);  // grkan_capi.cu

namespace {

template <typename T, bool EXACT, int MM1, int MN, bool FIXED>
__global__ void __launch_bounds__(256)
    k_bwd_terms(const T* __restrict__ x, const T* __restrict__ dy, T* __restrict__ dx,
                typename VecIO<T, 1>::A* __restrict__ terms, const typename VecIO<T, 1>::A* __restrict__ ca,
                const typename VecIO<T, 1>::A* __restrict__ cb, int64_t total, int d, int dg, int m1, int n) {
  using A = typename VecIO<T, 1>::A;
  using IO = VecIO<T, 1>;
  using Rat = Rational<A, EXACT, MM1, MN, FIXED>;
  Rat rat;
  int g_loaded = -1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int g = static_cast<int>(i % d) / dg;
    if (g != g_loaded) {
      rat.load(ca, cb, g, m1, n);
      g_loaded = g;
    }
    A vx[1], vu[1], o[1];
    IO::load(x + i, vx);
    IO::load(dy + i, vu);
    A acc[Rat::KC];
#pragma unroll
    for (int k = 0; k < Rat::KC; ++k) acc[k] = A(-0.0);
    o[0] = rat.grad(vx[0], vu[0], acc);
    IO::store(dx + i, o);
    for (int k = 0; k < m1; ++k) terms[k * total + i] = acc[k];
    for (int j = 0; j < n; ++j) terms[(m1 + j) * total + i] = acc[MM1 + j];
  }
}

template <typename T>
cudaError_t launch_terms(const void* x, const void* dy, void* dx, void* terms, const void* a, const void* b,
                         int64_t total, int d, int dg, int m1, int n, bool exact, cudaStream_t s) {
  using A = typename VecIO<T, 1>::A;
  const unsigned grid = static_cast<unsigned>(total / 256 + 1 < 148 * 16 ? total / 256 + 1 : 148 * 16);
  const bool fixed = m1 == 6 && n == 4;
  auto go = [&](auto kern) {
    kern<<<grid, 256, 0, s>>>(static_cast<const T*>(x), static_cast<const T*>(dy), static_cast<T*>(dx),
                              static_cast<A*>(terms), static_cast<const A*>(a), static_cast<const A*>(b), total, d,
                              dg, m1, n);
    return cudaGetLastError();
  };
  if (exact)
    return fixed ? go(k_bwd_terms<T, true, 6, 4, true>) : go(k_bwd_terms<T, true, 12, 12, false>);
  return fixed ? go(k_bwd_terms<T, false, 6, 4, true>) : go(k_bwd_terms<T, false, 12, 12, false>);
}

}  // namespace
}  // namespace grkan

extern "C" int grkan_bwd_terms(const void* x, const void* dy, const void* a, const void* b, void* dx, void* terms,
                               int64_t rows, int32_t d, int32_t n_groups, int32_t m1, int32_t n, int32_t dtype,
                               uint32_t flags, void* stream) {
  if (d < 1 || n_groups < 1 || d % n_groups)
    return grkan::set_error(GRKAN_ERR_LAYOUT, "layout mismatch: feature_dim not divisible by num_groups");
  if (rows < 0) return grkan::set_error(GRKAN_ERR_GRID, "grid geometry invalid: negative row count");
  if (m1 < 1 || n < 0 || m1 > GRKAN_MAX_M1 || n > GRKAN_MAX_N)
    return grkan::set_error(GRKAN_ERR_UNSUPPORTED, "degrees outside this build");
  if (flags & ~(GRKAN_FLAG_EXACT)) return grkan::set_error(GRKAN_ERR_INVALID, "unknown flag bits");
  if (rows == 0) return GRKAN_OK;
  if (!x || !dy || !dx || !terms || !a || (n > 0 && !b)) return grkan::set_error(GRKAN_ERR_INVALID, "null pointer");
  const int64_t total = rows * d;
  const bool exact = (flags & GRKAN_FLAG_EXACT) != 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  switch (dtype) {
    case GRKAN_F32: e = grkan::launch_terms<float>(x, dy, dx, terms, a, b, total, d, d / n_groups, m1, n, exact, s); break;
    case GRKAN_F64: e = grkan::launch_terms<double>(x, dy, dx, terms, a, b, total, d, d / n_groups, m1, n, exact, s); break;
    case GRKAN_BF16:
      e = grkan::launch_terms<__nv_bfloat16>(x, dy, dx, terms, a, b, total, d, d / n_groups, m1, n, exact, s);
      break;
    default: return grkan::set_error(GRKAN_ERR_UNSUPPORTED, "unsupported dtype");
  }
  if (e != cudaSuccess) return grkan::set_error(GRKAN_ERR_CUDA, cudaGetErrorString(e));
  return GRKAN_OK;
}
