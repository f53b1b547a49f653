// grkan_kernels.cuh -- the GR-KAN hot-path kernels for sm_100a.
//
//   K1 k_fwd          y = P(x)/Q(x)                      (forward_tensor, rational.py:325-345)
//   K2 k_bwd_main     dx + one partial per (row tile, group) per coefficient, no atomics
//                     (gradient_terms + block_partial_totals + _blocked_group_chunk,
//                      rational.py:227-278, backward.py:122-139, 249-272)
//   K3 k_bwd_reduce   fixed-order fp64 fold of the partials -> da, db; overflow flag
//                     (combine_partials + _check_accumulators, backward.py:142-184)
//   K4 k_bwd_atomic   the paper's Alg. 1 (per-element atomicAdd) -- comparator only
//                     (backward_naive as its model, backward.py:187-246)
//
// Work decomposition (shared by K1/K2/K4).  The tensor is [rows, d] row-major;
// group g owns columns [g*dg, (g+1)*dg).  One CTA owns one (row tile, group):
// R rows x dg columns, so its coefficients are CTA-uniform registers and its
// coefficient gradients reduce to exactly one partial.  Linear CTA id
// = tile * n_groups + g, so CTAs resident together stream one contiguous row
// band.  Inside a CTA, thread (tr, tc) owns vector column tc (+CT, ...) and rows
// tr, tr+RPB, ...; a warp covers consecutive 16-byte vectors of a row segment,
// i.e. fully coalesced 128-bit loads and stores.  U row-vectors are loaded
// before any math so each thread keeps 2*U 16-byte loads in flight.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

#include "grkan_math.cuh"

namespace grkan {

struct Geom {
  int64_t rows;     // B*L
  int64_t n_tiles;  // ceil(rows / R)
  int32_t d;        // feature dim (row stride, elements)
  int32_t ng;       // groups
  int32_t dg;       // group width
  int32_t V;        // vectors per row segment = dg / W
  int32_t CT;       // threads along vector columns
  int32_t RPB;      // threads along rows; blockDim = CT * RPB
  int32_t R;        // rows per tile (multiple of RPB * U)
};

struct DevStatus {
  int32_t nonfinite_input;
  int32_t accum_overflow;
};

// ---------------------------------------------------------------------------
// Vector I/O: W elements of T <-> accumulation type A.  Streaming (.cs) hints:
// every byte is touched once per kernel, keep it from displacing L2.
// ---------------------------------------------------------------------------
template <typename T, int W>
struct VecIO;

template <>
struct VecIO<float, 4> {
  using A = float;
  static __device__ __forceinline__ void load(const float* p, A (&v)[4]) {
    const float4 t = __ldcs(reinterpret_cast<const float4*>(p));
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  }
  static __device__ __forceinline__ void store(float* p, const A (&v)[4]) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
  }
};

template <>
struct VecIO<float, 1> {
  using A = float;
  static __device__ __forceinline__ void load(const float* p, A (&v)[1]) { v[0] = __ldcs(p); }
  static __device__ __forceinline__ void store(float* p, const A (&v)[1]) { __stcs(p, v[0]); }
};

template <>
struct VecIO<double, 2> {
  using A = double;
  static __device__ __forceinline__ void load(const double* p, A (&v)[2]) {
    const double2 t = __ldcs(reinterpret_cast<const double2*>(p));
    v[0] = t.x; v[1] = t.y;
  }
  static __device__ __forceinline__ void store(double* p, const A (&v)[2]) {
    __stcs(reinterpret_cast<double2*>(p), make_double2(v[0], v[1]));
  }
};

template <>
struct VecIO<double, 1> {
  using A = double;
  static __device__ __forceinline__ void load(const double* p, A (&v)[1]) { v[0] = __ldcs(p); }
  static __device__ __forceinline__ void store(double* p, const A (&v)[1]) { __stcs(p, v[0]); }
};

// bf16: 8 elements per 16-byte vector; widening is a shift / mask per element,
// narrowing is one round-to-nearest-even pack per pair.
template <>
struct VecIO<__nv_bfloat16, 8> {
  using A = float;
  static __device__ __forceinline__ void load(const __nv_bfloat16* p, A (&v)[8]) {
    const uint4 t = __ldcs(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
  static __device__ __forceinline__ void store(__nv_bfloat16* p, const A (&v)[8]) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
      w[i] = *reinterpret_cast<const uint32_t*>(&h);
    }
    __stcs(reinterpret_cast<uint4*>(p), make_uint4(w[0], w[1], w[2], w[3]));
  }
};

template <>
struct VecIO<__nv_bfloat16, 1> {
  using A = float;
  static __device__ __forceinline__ void load(const __nv_bfloat16* p, A (&v)[1]) {
    const unsigned short h = __ldcs(reinterpret_cast<const unsigned short*>(p));
    v[0] = __uint_as_float(static_cast<uint32_t>(h) << 16);
  }
  static __device__ __forceinline__ void store(__nv_bfloat16* p, const A (&v)[1]) {
    const __nv_bfloat16 h = __float2bfloat16_rn(v[0]);
    __stcs(reinterpret_cast<unsigned short*>(p), *reinterpret_cast<const unsigned short*>(&h));
  }
};

template <typename A>
__device__ __forceinline__ bool nonfinite(A v) {
  return !(fabs(v) <= (sizeof(A) == 4 ? A(FLT_MAX) : A(DBL_MAX)));
}

__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

constexpr int kMaxThreads = 512;

// Unrolled row-vectors per thread per step.
template <int W>
struct Unroll {
  static constexpr int U = W >= 8 ? 2 : 4;
};

// ---------------------------------------------------------------------------
// Tile walker: calls body(elem_offset, valid) for the U row-vectors of each
// step; the common full-tile case is branch-free.
// ---------------------------------------------------------------------------
struct TileCtx {
  int64_t row0;
  int nr;
  int tc, tr;
};

__device__ __forceinline__ TileCtx tile_ctx(const Geom& geo, int64_t tile) {
  TileCtx t;
  t.row0 = tile * geo.R;
  const int64_t left = geo.rows - t.row0;
  t.nr = left < geo.R ? static_cast<int>(left) : geo.R;
  t.tc = threadIdx.x % geo.CT;
  t.tr = threadIdx.x / geo.CT;
  return t;
}

// ---------------------------------------------------------------------------
// K1: forward
// ---------------------------------------------------------------------------
template <typename T, bool EXACT, int MM1, int MN, bool FIXED, int W>
__global__ void __launch_bounds__(kMaxThreads, 1)
    k_fwd(const T* __restrict__ x, T* __restrict__ y, const typename VecIO<T, W>::A* __restrict__ ca,
          const typename VecIO<T, W>::A* __restrict__ cb, Geom geo, int m1, int n, int check,
          DevStatus* __restrict__ st) {
  using A = typename VecIO<T, W>::A;
  using IO = VecIO<T, W>;
  constexpr int U = Unroll<W>::U;
  const int64_t bid = blockIdx.x;
  const int g = static_cast<int>(bid % geo.ng);
  const int64_t tile = bid / geo.ng;
  Rational<A, EXACT, MM1, MN, FIXED> rat;
  rat.load(ca, cb, g, m1, n);
  const TileCtx tc = tile_ctx(geo, tile);
  bool bad = false;
  for (int c = tc.tc; c < geo.V; c += geo.CT) {
    const int64_t base = (tc.row0 * geo.d) + (int64_t)g * geo.dg + (int64_t)c * W;
    for (int r = tc.tr; r < tc.nr; r += geo.RPB * U) {
      A v[U][W];
      const bool full = r + (U - 1) * geo.RPB < tc.nr;
#pragma unroll
      for (int j = 0; j < U; ++j) {
        if (full || r + j * geo.RPB < tc.nr) IO::load(x + base + (int64_t)(r + j * geo.RPB) * geo.d, v[j]);
      }
#pragma unroll
      for (int j = 0; j < U; ++j) {
        if (full || r + j * geo.RPB < tc.nr) {
          A o[W];
#pragma unroll
          for (int e = 0; e < W; ++e) {
            if (check) bad |= nonfinite(v[j][e]);
            o[e] = rat.value(v[j][e]);
          }
          IO::store(y + base + (int64_t)(r + j * geo.RPB) * geo.d, o);
        }
      }
    }
  }
  if (check && bad) st->nonfinite_input = 1;  // plain store of a constant: no atomic needed
}

// ---------------------------------------------------------------------------
// Deterministic CTA reduction of KC per-thread accumulators -> one partial.
// Warp butterfly, then warp 0 folds the per-warp sums in warp order.
// Partials are stored SoA: part[(g*KC + k) * n_tiles + tile].
// ---------------------------------------------------------------------------
template <typename A, int KC>
__device__ __forceinline__ void cta_reduce_store(A (&acc)[KC], int kc_rt, A* __restrict__ part,
                                                 int g, int64_t tile, int64_t n_tiles) {
  __shared__ A red[kMaxThreads / 32][KC];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    A v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][k] = v;
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < KC; ++k) {
      A v = lane < nwarps ? red[lane][k] : A(0);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && k < kc_rt) part[((int64_t)g * kc_rt + k) * n_tiles + tile] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// K2: backward main pass
// ---------------------------------------------------------------------------
template <typename T, bool EXACT, int MM1, int MN, bool FIXED, int W>
__global__ void __launch_bounds__(kMaxThreads, 1)
    k_bwd_main(const T* __restrict__ x, const T* __restrict__ dy, T* __restrict__ dx,
               const typename VecIO<T, W>::A* __restrict__ ca,
               const typename VecIO<T, W>::A* __restrict__ cb,
               typename VecIO<T, W>::A* __restrict__ part, Geom geo, int m1, int n, int check,
               DevStatus* __restrict__ st) {
  using A = typename VecIO<T, W>::A;
  using IO = VecIO<T, W>;
  using Rat = Rational<A, EXACT, MM1, MN, FIXED>;
  constexpr int U = Unroll<W>::U;
  constexpr int KC = Rat::KC;
  // Let K3 (launched with programmatic stream serialization) get scheduled;
  // it waits in griddepcontrol.wait until this grid has fully completed.
  pdl_launch_dependents();
  const int64_t bid = blockIdx.x;
  const int g = static_cast<int>(bid % geo.ng);
  const int64_t tile = bid / geo.ng;
  Rat rat;
  rat.load(ca, cb, g, m1, n);
  A acc[KC];
#pragma unroll
  for (int k = 0; k < KC; ++k) acc[k] = A(0);
  const TileCtx tc = tile_ctx(geo, tile);
  bool bad = false;
  for (int c = tc.tc; c < geo.V; c += geo.CT) {
    const int64_t base = (tc.row0 * geo.d) + (int64_t)g * geo.dg + (int64_t)c * W;
    for (int r = tc.tr; r < tc.nr; r += geo.RPB * U) {
      A vx[U][W], vu[U][W];
      const bool full = r + (U - 1) * geo.RPB < tc.nr;
#pragma unroll
      for (int j = 0; j < U; ++j) {
        if (full || r + j * geo.RPB < tc.nr) {
          const int64_t off = base + (int64_t)(r + j * geo.RPB) * geo.d;
          IO::load(x + off, vx[j]);
          IO::load(dy + off, vu[j]);
        }
      }
#pragma unroll
      for (int j = 0; j < U; ++j) {
        if (full || r + j * geo.RPB < tc.nr) {
          A o[W];
#pragma unroll
          for (int e = 0; e < W; ++e) {
            if (check) bad |= nonfinite(vx[j][e]) | nonfinite(vu[j][e]);
            o[e] = rat.grad(vx[j][e], vu[j][e], acc);
          }
          IO::store(dx + base + (int64_t)(r + j * geo.RPB) * geo.d, o);
        }
      }
    }
  }
  if (check && bad) st->nonfinite_input = 1;
  cta_reduce_store<A, KC>(acc, rat.m1 + rat.n, part, g, tile, geo.n_tiles);
}

// ---------------------------------------------------------------------------
// K3: fixed-order reduction of the partials, one CTA per (group, coefficient).
// fp64 accumulation; thread t folds tiles t, t+B, ... in order, then a fixed
// butterfly / warp-order tree.  Bitwise reproducible for a given geometry.
// ---------------------------------------------------------------------------
template <typename A>
__global__ void __launch_bounds__(256)
    k_bwd_reduce(const A* __restrict__ part, int64_t n_tiles, int m1, int n, A* __restrict__ da,
                 A* __restrict__ db, DevStatus* __restrict__ st) {
  pdl_wait();  // K2's partials are complete and visible after this
  const int kc = m1 + n;
  const int col = blockIdx.x;  // g * kc + k
  const A* src = part + (int64_t)col * n_tiles;
  double s = 0.0;
  for (int64_t t = threadIdx.x; t < n_tiles; t += blockDim.x) s += static_cast<double>(src[t]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ double red[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    const int nw = (blockDim.x + 31) >> 5;
    for (int w = 0; w < nw; ++w) tot += red[w];
    const A out = static_cast<A>(tot);
    const int g = col / kc, k = col % kc;
    if (k < m1)
      da[(int64_t)g * m1 + k] = out;
    else
      db[(int64_t)g * n + (k - m1)] = out;
    if (nonfinite(out)) st->accum_overflow = 1;
  }
}

// ---------------------------------------------------------------------------
// K4: Alg. 1 comparator -- every element atomically adds its m1+n terms.
// ---------------------------------------------------------------------------
template <typename T, bool EXACT, int MM1, int MN, bool FIXED, int W>
__global__ void __launch_bounds__(kMaxThreads, 1)
    k_bwd_atomic(const T* __restrict__ x, const T* __restrict__ dy, T* __restrict__ dx,
                 const typename VecIO<T, W>::A* __restrict__ ca,
                 const typename VecIO<T, W>::A* __restrict__ cb, typename VecIO<T, W>::A* da,
                 typename VecIO<T, W>::A* db, Geom geo, int m1, int n) {
  using A = typename VecIO<T, W>::A;
  using IO = VecIO<T, W>;
  using Rat = Rational<A, EXACT, MM1, MN, FIXED>;
  constexpr int KC = Rat::KC;
  const int64_t bid = blockIdx.x;
  const int g = static_cast<int>(bid % geo.ng);
  const int64_t tile = bid / geo.ng;
  Rat rat;
  rat.load(ca, cb, g, m1, n);
  const TileCtx tc = tile_ctx(geo, tile);
  for (int c = tc.tc; c < geo.V; c += geo.CT) {
    const int64_t base = (tc.row0 * geo.d) + (int64_t)g * geo.dg + (int64_t)c * W;
    for (int r = tc.tr; r < tc.nr; r += geo.RPB) {
      const int64_t off = base + (int64_t)r * geo.d;
      A vx[W], vu[W], o[W];
      IO::load(x + off, vx);
      IO::load(dy + off, vu);
#pragma unroll
      for (int e = 0; e < W; ++e) {
        A t[KC];
#pragma unroll
        for (int k = 0; k < KC; ++k) t[k] = A(0);
        o[e] = rat.grad(vx[e], vu[e], t);
#pragma unroll
        for (int i = 0; i < MM1; ++i)
          if (FIXED || i < rat.m1) atomicAdd(da + (int64_t)g * rat.m1 + i, t[i]);
#pragma unroll
        for (int j = 0; j < MN; ++j)
          if (FIXED || j < rat.n) atomicAdd(db + (int64_t)g * rat.n + j, t[MM1 + j]);
      }
      IO::store(dx + off, o);
    }
  }
}

// Overflow check for K4's outputs (one thread per coefficient).
template <typename A>
__global__ void k_check_finite(const A* __restrict__ v, int64_t cnt, DevStatus* __restrict__ st) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < cnt && nonfinite(v[i])) st->accum_overflow = 1;
}

}  // namespace grkan
