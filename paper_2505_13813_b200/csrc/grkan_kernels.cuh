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
// Work decomposition (K1/K2/K4).  The tensor is [rows, d] row-major; group g
// owns columns [g*dg, (g+1)*dg).  One CTA owns one (row tile, group) block of
// R rows x dg columns, so its coefficients are CTA-uniform registers and its
// coefficient gradients reduce to exactly one partial.  Linear CTA id
// = tile * n_groups + g, so CTAs resident together stream one contiguous row
// band.  Inside the tile the R x V grid of 16-byte vectors is walked in flat
// order by kBlock threads (thread t takes vectors t, t + kBlock, ...), so a
// warp always reads 32 consecutive vectors of a row segment: coalesced
// 128-bit loads/stores whatever the group width.  U vectors per tensor are
// loaded before any math, giving 2*U 16-byte loads in flight per thread.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

#include <type_traits>

#include "grkan_math.cuh"
#include "grkan_types.h"

namespace grkan {

// ---------------------------------------------------------------------------
// Vector I/O: W elements of T <-> math type A.  Streaming (.cs) hints: every
// byte is touched once per kernel, so keep it from displacing L2.
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
// narrowing one round-to-nearest-even pack per pair (F2FP.BF16.F32.PACK_AB).
template <>
struct VecIO<__nv_bfloat16, 8> {
  using A = float;
  static __device__ __forceinline__ void load(const __nv_bfloat16* p, A (&v)[8]) {
    const uint4 t = __ldcs(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(__byte_perm(w[i], 0u, 0x1044));  // w << 16 on the ALU pipe (PRMT)
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

// FAST sign guard per I/O type (RationalX2::grad_n): on for fp32, off for bf16.
template <typename T>
constexpr bool kGuard = GRKAN_BF16_GUARD || !std::is_same<T, __nv_bfloat16>::value;

__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Diagnostic only (GRKAN_PROBE_TIMES=1 variant builds, tools/probe_times.py):
// %globaltimer stamps per staged-backward CTA [start, first stage, warp 0 done,
// last warp done] and K3's [first start, last end] after them.
#if GRKAN_PROBE_TIMES
constexpr int kProbeCtas = 4096;
static __device__ unsigned long long g_probe_t[4 * kProbeCtas + 4];
__device__ __forceinline__ unsigned long long probe_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define GRKAN_STAMP(i) (g_probe_t[4 * (blockIdx.x % kProbeCtas) + (i)] = probe_now())
#define GRKAN_STAMP_MAX(i) atomicMax(&g_probe_t[4 * (blockIdx.x % kProbeCtas) + (i)], probe_now())
#define GRKAN_PROBE_EXPORTS(SUF)                                                              \
  extern "C" __attribute__((visibility("default"))) int grkan_probe_read_##SUF(unsigned long long* h, int n) {                      \
    return (int)cudaMemcpyFromSymbol(h, grkan::g_probe_t, sizeof(unsigned long long) * n);  \
  }                                                                                           \
  extern "C" __attribute__((visibility("default"))) int grkan_probe_clear_##SUF() {                                                 \
    static unsigned long long z[4 * grkan::kProbeCtas + 4];                                   \
    z[4 * grkan::kProbeCtas] = ~0ull; /* K3's first start: atomicMin */                        \
    return (int)cudaMemcpyToSymbol(grkan::g_probe_t, z, sizeof(z));                         \
  }
#else
#define GRKAN_STAMP(i) ((void)0)
#define GRKAN_STAMP_MAX(i) ((void)0)
#define GRKAN_PROBE_EXPORTS(SUF)
#endif

// ---------------------------------------------------------------------------
// Engine selection: packed fp32 pairs for the paper's degrees, scalar otherwise.
// ---------------------------------------------------------------------------
template <typename T, bool EXACT, int MM1, int MN, bool FIXED, int W>
struct Engine {
  using A = typename VecIO<T, W>::A;
  static constexpr bool kPacked = std::is_same<A, float>::value && FIXED &&
                                  ((MM1 == 6 && MN == 4) || (MM1 == 4 && MN == 2)) && (W % 2 == 0);
  using Scalar = Rational<A, EXACT, MM1, MN, FIXED>;
  using Packed = RationalX2<EXACT, kPacked ? MM1 : 6, kPacked ? MN : 4>;
  static constexpr int KC = MM1 + MN;
  // vectors per tensor per thread per step (backward; = unroll_for_width(W))
  static constexpr int U = W >= 2 ? 2 : 4;
  // forward: one tensor in and little math per byte, so more loads in flight
  static constexpr int UF = 4;
};

// Flat walk of one tile: the thread's current (row, vector) position.
struct Cursor {
  int r, c;
  __device__ __forceinline__ void init(int k, int V) {
    r = k / V;
    c = k - r * V;
  }
  __device__ __forceinline__ void advance(const Geom& g) {
    c += g.dc;
    r += g.dr;
    if (c >= g.V) {
      c -= g.V;
      ++r;
    }
  }
};

// NaN / Inf detector for checked mode: x * 0 is NaN exactly when x is not finite.
template <typename A>
struct Checker {
  A acc = A(0);
  __device__ __forceinline__ void add(A v) { acc = fma(v, A(0), acc); }
  __device__ __forceinline__ bool bad() const { return nonfinite(acc); }
};

// ---------------------------------------------------------------------------
// Access instrumentation (INSTR instantiations only; the reference's counter= and
// coverage= arguments, pkg/src/grkan/backward.py:187-195,275-285,326-351).  Every
// element a thread processes bumps its coverage cell; each thread tallies the
// element-sized global accesses it performs, in the reference's units (one load or
// store = 1; an atomic add = 1 read + 1 write + 1 rmw), flushed once per warp.
// ---------------------------------------------------------------------------
struct Tally {
  unsigned long long r = 0, w = 0, m = 0;
  __device__ __forceinline__ void flush(const Geom& geo) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      r += __shfl_xor_sync(0xffffffffu, r, o);
      w += __shfl_xor_sync(0xffffffffu, w, o);
      m += __shfl_xor_sync(0xffffffffu, m, o);
    }
    if ((threadIdx.x & 31) == 0) {
      if (r) atomicAdd(geo.cnt + 0, r);
      if (w) atomicAdd(geo.cnt + 1, w);
      if (m) atomicAdd(geo.cnt + 2, m);
    }
  }
};
template <int W>
__device__ __forceinline__ void visit(const Geom& geo, int64_t elem_off) {
#pragma unroll
  for (int e = 0; e < W; ++e) atomicAdd(geo.cov + elem_off + e, 1);
}

// ---------------------------------------------------------------------------
// K1: forward
// ---------------------------------------------------------------------------
template <typename T, bool EXACT, int MM1, int MN, bool FIXED, int W, bool CHECK>
__global__ void __launch_bounds__(kBlock, kMinBlocks)
    k_fwd(const T* __restrict__ x, T* __restrict__ y,
          const typename VecIO<T, W>::A* __restrict__ ca,
          const typename VecIO<T, W>::A* __restrict__ cb, Geom geo, int m1, int n,
          DevStatus* __restrict__ st) {
  using E = Engine<T, EXACT, MM1, MN, FIXED, W>;
  using A = typename E::A;
  using IO = VecIO<T, W>;
  constexpr int U = E::UF;
  const int64_t bid = blockIdx.x;
  const int g = static_cast<int>(bid % geo.ng);
  const int64_t tile = bid / geo.ng;
  typename E::Scalar rs;
  typename E::Packed rp;
  if constexpr (E::kPacked) rp.load(ca, cb, g, geo.one); else rs.load(ca, cb, g, m1, n);
  const int64_t row0 = tile * geo.R;
  const int nr = static_cast<int>(geo.rows - row0 < geo.R ? geo.rows - row0 : geo.R);
  const int nvec = nr * geo.V;
  const int64_t tile_off = row0 * geo.d + (int64_t)g * geo.dg;
  const T* xt = x + tile_off;
  T* yt = y + tile_off;
  Checker<A> chk;
  Cursor cur;
  cur.init(threadIdx.x, geo.V);
  for (int k = threadIdx.x; k < nvec; k += U * kBlock) {
    int64_t off[U];
    A v[U][W];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      off[j] = (int64_t)cur.r * geo.d + cur.c * W;
      cur.advance(geo);
    }
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (j == 0 || k + j * kBlock < nvec) IO::load(xt + off[j], v[j]);
#pragma unroll
    for (int j = 0; j < U; ++j) {
      if (j == 0 || k + j * kBlock < nvec) {
        A o[W];
        if constexpr (E::kPacked) {
#pragma unroll
          for (int e = 0; e < W; e += 2) {
            const float2 r2 = rp.value(make_float2(v[j][e], v[j][e + 1]));
            o[e] = r2.x;
            o[e + 1] = r2.y;
          }
        } else {
#pragma unroll
          for (int e = 0; e < W; ++e) o[e] = rs.value(v[j][e]);
        }
        if constexpr (CHECK) {
#pragma unroll
          for (int e = 0; e < W; ++e) chk.add(v[j][e]);
        }
        IO::store(yt + off[j], o);
      }
    }
  }
  if (CHECK && chk.bad()) st->nonfinite_input = 1;  // plain store of a constant: no atomic
}

// ---------------------------------------------------------------------------
// Deterministic CTA reduction of the accumulators -> one partial per slot.
// Warp butterfly (fixed), then warp 0 folds the per-warp sums in warp order.
// Partials are SoA: part[(g * kc + k) * n_tiles + tile], k in [0, m1 + n):
// slot k < m1 is a_k's term, slot m1 + j is b_{j+1}'s (accumulator MM1 + j).
// ---------------------------------------------------------------------------
template <typename A, int MM1, int KC>
__device__ __forceinline__ void cta_reduce_store(A (&acc)[KC], int m1, int n, A* __restrict__ part,
                                                 int g, int64_t tile, int64_t n_tiles, int ng, bool det) {
  __shared__ A red[kBlock / 32][KC];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    A v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][k] = v;
  }
  __syncthreads();
  if (warp == 0) {
    const int kc = m1 + n;
#pragma unroll
    for (int k = 0; k < KC; ++k) {
      A v = lane < kBlock / 32 ? red[lane][k] : A(0);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      const bool live = k < MM1 ? (k < m1) : (k - MM1 < n);
      const int slot = k < MM1 ? k : m1 + (k - MM1);
      if (lane == 0 && live)
        part[det ? (tile * ng + g) * kc + slot : ((int64_t)g * kc + slot) * n_tiles + tile] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// K2: backward main pass
// ---------------------------------------------------------------------------
template <typename T, bool EXACT, int MM1, int MN, bool FIXED, int W, bool CHECK, bool INSTR = false>
__global__ void __launch_bounds__(kBlock, kMinBlocks)
    k_bwd_main(const T* __restrict__ x, const T* __restrict__ dy, T* __restrict__ dx,
               const typename VecIO<T, W>::A* __restrict__ ca,
               const typename VecIO<T, W>::A* __restrict__ cb,
               typename VecIO<T, W>::A* __restrict__ part, Geom geo, int m1, int n,
               DevStatus* __restrict__ st) {
  using E = Engine<T, EXACT, MM1, MN, FIXED, W>;
  using A = typename E::A;
  using IO = VecIO<T, W>;
  constexpr int U = E::U;
  constexpr int KC = E::KC;
  // Let K3 (launched with programmatic stream serialization) get scheduled;
  // it waits in griddepcontrol.wait until this whole grid has completed.
  pdl_launch_dependents();
  const int64_t bid = blockIdx.x;
  const int g = static_cast<int>(bid % geo.ng);
  const int64_t tile = bid / geo.ng;
  typename E::Scalar rs;
  typename E::Packed rp;
  A acc[KC];
  float2 acc2[E::kPacked ? KC : 1];
  if constexpr (E::kPacked) {
    rp.load(ca, cb, g, geo.one);
#pragma unroll
    for (int k = 0; k < KC; ++k) acc2[k] = make_float2(0.f, 0.f);
  } else {
    rs.load(ca, cb, g, m1, n);
#pragma unroll
    for (int k = 0; k < KC; ++k) acc[k] = A(0);
  }
  const int64_t row0 = tile * geo.R;
  const int nr = static_cast<int>(geo.rows - row0 < geo.R ? geo.rows - row0 : geo.R);
  const int nvec = nr * geo.V;
  const int64_t tile_off = row0 * geo.d + (int64_t)g * geo.dg;
  const T* xt = x + tile_off;
  const T* ut = dy + tile_off;
  T* dt = dx + tile_off;
  Checker<A> chk;
  Tally tl;
  Cursor cur;
  cur.init(threadIdx.x, geo.V);
  for (int k = threadIdx.x; k < nvec; k += U * kBlock) {
    int64_t off[U];
    A vx[U][W], vu[U][W];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      off[j] = (int64_t)cur.r * geo.d + cur.c * W;
      cur.advance(geo);
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      if (j == 0 || k + j * kBlock < nvec) {
        IO::load(xt + off[j], vx[j]);
        IO::load(ut + off[j], vu[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      if (j == 0 || k + j * kBlock < nvec) {
        A o[W];
        if constexpr (E::kPacked) {
rp.template grad_n<W / 2, kGuard<T>>(vx[j], vu[j], o, acc2);
        } else {
#pragma unroll
          for (int e = 0; e < W; ++e) o[e] = rs.grad(vx[j][e], vu[j][e], acc);
        }
        if constexpr (CHECK) {
#pragma unroll
          for (int e = 0; e < W; ++e) {
            chk.add(vx[j][e]);
            chk.add(vu[j][e]);
          }
        }
        IO::store(dt + off[j], o);
        if constexpr (INSTR) {
          visit<W>(geo, tile_off + off[j]);
          tl.r += 2 * W;  // x, dy
          tl.w += W;      // dx
        }
      }
    }
  }
  if (CHECK && chk.bad()) st->nonfinite_input = 1;
  if constexpr (INSTR) {
    if (threadIdx.x == 0) {
      const int kc = FIXED ? MM1 + MN : m1 + n;
      tl.r += kc;  // the CTA's coefficient row (held in registers afterwards)
      tl.w += kc;  // its one partial per coefficient
    }
    tl.flush(geo);
  }
  if constexpr (E::kPacked) {
#pragma unroll
    for (int k = 0; k < KC; ++k) acc[k] = acc2[k].x + acc2[k].y;
    cta_reduce_store<A, MM1, KC>(acc, MM1, MN, part, g, tile, geo.n_tiles, geo.ng, geo.det != 0);
  } else {
    cta_reduce_store<A, MM1, KC>(acc, FIXED ? MM1 : m1, FIXED ? MN : n, part, g, tile, geo.n_tiles, geo.ng, geo.det != 0);
  }
}

// ---------------------------------------------------------------------------
// K3: fixed-order reduction of the partials, one CTA per (group, coefficient).
// fp64 accumulation; thread t folds tiles t, t+B, ... in order, then a fixed
// butterfly / warp-order tree.  Bitwise reproducible for a given geometry.
// ---------------------------------------------------------------------------
template <typename A>
__global__ void __launch_bounds__(256)
    k_bwd_reduce(const A* __restrict__ part, int64_t n_tiles, int m1, int n, A* __restrict__ da,
                 A* __restrict__ db, DevStatus* __restrict__ st, int64_t slot_stride,
                 unsigned long long* __restrict__ cnt) {
  pdl_wait();  // K2's partials are complete and visible after this
#if GRKAN_PROBE_TIMES
  if (threadIdx.x == 0) atomicMin(&g_probe_t[4 * kProbeCtas], probe_now());
#endif
  const int kc = m1 + n;
  const int col = blockIdx.x;  // g * kc + k
  // column-major part[col * n_tiles + t] (slot_stride 1), or the deterministic
  // mode's slot-major part[t * ng * kc + col] (slot_stride ng * kc)
  const A* src = part + (slot_stride == 1 ? (int64_t)col * n_tiles : (int64_t)col);
  double s = 0.0;
  for (int64_t t = threadIdx.x; t < n_tiles; t += blockDim.x) s += static_cast<double>(src[t * slot_stride]);
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
#if GRKAN_PROBE_TIMES
    atomicMax(&g_probe_t[4 * kProbeCtas + 1], probe_now());
#endif
    if (cnt) {  // instrumented: this column's partial loads and its one result store
      atomicAdd(cnt + 0, static_cast<unsigned long long>(n_tiles));
      atomicAdd(cnt + 1, 1ull);
    }
  }
}

// ---------------------------------------------------------------------------
// K4: Alg. 1 comparator -- every element atomically adds its m1+n terms.
// ---------------------------------------------------------------------------
template <typename T, bool EXACT, int MM1, int MN, bool FIXED, int W, bool INSTR = false>
__global__ void __launch_bounds__(kBlock)
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
  const int64_t row0 = tile * geo.R;
  const int nr = static_cast<int>(geo.rows - row0 < geo.R ? geo.rows - row0 : geo.R);
  const int nvec = nr * geo.V;
  const int64_t tile_off = row0 * geo.d + (int64_t)g * geo.dg;
  Tally tl;
  Cursor cur;
  cur.init(threadIdx.x, geo.V);
  for (int k = threadIdx.x; k < nvec; k += kBlock) {
    const int64_t off = tile_off + (int64_t)cur.r * geo.d + cur.c * W;
    cur.advance(geo);
    A vx[W], vu[W], o[W];
    IO::load(x + off, vx);
    IO::load(dy + off, vu);
#pragma unroll
    for (int e = 0; e < W; ++e) {
      A t[KC];
#pragma unroll
      for (int i = 0; i < KC; ++i) t[i] = A(0);
      o[e] = rat.grad(vx[e], vu[e], t);
#pragma unroll
      for (int i = 0; i < MM1; ++i)
        if (FIXED || i < rat.m1) atomicAdd(da + (int64_t)g * rat.m1 + i, t[i]);
#pragma unroll
      for (int j = 0; j < MN; ++j)
        if (FIXED || j < rat.n) atomicAdd(db + (int64_t)g * rat.n + j, t[MM1 + j]);
    }
    IO::store(dx + off, o);
    if constexpr (INSTR) {
      visit<W>(geo, off);
      const unsigned long long kc = FIXED ? MM1 + MN : rat.m1 + rat.n;
      tl.r += W * (2 + kc);  // x, dy, and the read half of each coefficient atomic
      tl.w += W * (1 + kc);  // dx, and the write half
      tl.m += W * kc;
    }
  }
  if constexpr (INSTR) {
    if (threadIdx.x == 0) tl.r += FIXED ? MM1 + MN : rat.m1 + rat.n;  // the CTA's coefficient row
    tl.flush(geo);
  }
}

// Overflow check for K4's outputs (one thread per coefficient).
template <typename A>
__global__ void k_check_finite(const A* __restrict__ v, int64_t cnt, DevStatus* __restrict__ st) {
  // grid-stride: any coefficient count (n_groups * (m + 1) is unbounded)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
    if (nonfinite(v[i])) st->accum_overflow = 1;
}

}  // namespace grkan
