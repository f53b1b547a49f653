// grkan_math.cuh -- per-element GR-KAN math for sm_100a, two precision policies.
//
// EXACT: the reference's operation order with every *, +, /, 1/q rounded on its
//        own (__fmul_rn / __fadd_rn / __fdiv_rn / __frcp_rn; the _rn intrinsics
//        are never contracted into FMA).  y, dx and each of the m1+n per-element
//        coefficient-gradient terms are then bitwise equal to the reference
//        (pkg/src/grkan/rational.py:195-278).
// FAST:  FMA Horner, one approximate reciprocal (Q >= 1 so rcp.approx is
//        safe), powers of x shared by the da and db terms.  Restructured but
//        algebraically identical; gated at max-scaled error <= 1e-5.
//
// Coefficients are CTA-uniform (one group per CTA) and live in registers.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace grkan {

// ---------------------------------------------------------------------------
// Scalar op policies
// ---------------------------------------------------------------------------
template <typename A, bool EXACT>
struct Op;

template <>
struct Op<float, true> {
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float mad(float a, float b, float c) {
    return __fadd_rn(__fmul_rn(a, b), c);
  }
  static __device__ __forceinline__ float rcp(float q) { return __frcp_rn(q); }
  static __device__ __forceinline__ float div(float p, float q) { return __fdiv_rn(p, q); }
};

template <>
struct Op<float, false> {
  static __device__ __forceinline__ float mul(float a, float b) { return a * b; }
  static __device__ __forceinline__ float add(float a, float b) { return a + b; }
  static __device__ __forceinline__ float sub(float a, float b) { return a - b; }
  static __device__ __forceinline__ float mad(float a, float b, float c) { return fmaf(a, b, c); }
  // q >= 1 always (safe Pade denominator), so the MUFU approximation has no
  // denormal corner; q = inf gives 0 like the IEEE path.
  static __device__ __forceinline__ float rcp(float q) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(q));
    return r;
  }
  static __device__ __forceinline__ float div(float p, float q) { return p * rcp(q); }
};

template <>
struct Op<double, true> {
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mad(double a, double b, double c) {
    return __dadd_rn(__dmul_rn(a, b), c);
  }
  static __device__ __forceinline__ double rcp(double q) { return __drcp_rn(q); }
  static __device__ __forceinline__ double div(double p, double q) { return __ddiv_rn(p, q); }
};

template <>
struct Op<double, false> {
  static __device__ __forceinline__ double mul(double a, double b) { return a * b; }
  static __device__ __forceinline__ double add(double a, double b) { return a + b; }
  static __device__ __forceinline__ double sub(double a, double b) { return a - b; }
  static __device__ __forceinline__ double mad(double a, double b, double c) { return fma(a, b, c); }
  static __device__ __forceinline__ double rcp(double q) { return 1.0 / q; }
  static __device__ __forceinline__ double div(double p, double q) { return p / q; }
};

// np.sign: +1 / -1 / +0 for +-0 / NaN propagates (rational.py:251)
template <typename A>
__device__ __forceinline__ A sign_of(A s) {
  return s > A(0) ? A(1) : (s < A(0) ? A(-1) : (s == A(0) ? A(0) : s));
}

// ---------------------------------------------------------------------------
// Horner with a compile-time (FIXED) or uniform run-time coefficient count.
// The run-time form never indexes registers dynamically: every step is
// computed and a uniform select keeps the right one, so the rounding sequence
// is exactly the reference's acc = c_top; acc = acc * x + c_k (rational.py:195-200).
// ---------------------------------------------------------------------------
template <typename A, bool EXACT, int MAXC, bool FIXED>
__device__ __forceinline__ A horner(const A (&c)[MAXC], int cnt, A x) {
  using O = Op<A, EXACT>;
  A acc = c[MAXC - 1];
#pragma unroll
  for (int k = MAXC - 2; k >= 0; --k) {
    const A t = O::mad(acc, x, c[k]);
    if (FIXED) {
      acc = t;
    } else {
      acc = (k == cnt - 1) ? c[k] : ((k < cnt - 1) ? t : acc);
    }
  }
  return acc;
}

// ---------------------------------------------------------------------------
// One coefficient row (one group), held in registers.
//   MM1 / MN: compile-time capacity; FIXED: m1 == MM1 and n == MN exactly.
// ---------------------------------------------------------------------------
template <typename A, bool EXACT, int MM1, int MN, bool FIXED>
struct Rational {
  static constexpr int KC = MM1 + MN;               // accumulator slots
  static constexpr int ND = MM1 > 1 ? MM1 - 1 : 1;  // numerator-derivative slots
  static constexpr int NB = MN > 0 ? MN : 1;

  A a[MM1];
  A b[NB];
  A da[ND];  // k * a_k, k = 1..m   (rational.py:203-208)
  A db[NB];  // k * b_k, k = 1..n   (derivative of [0, b], rational.py:255)
  int m1, n;

  __device__ __forceinline__ void load(const A* __restrict__ ga, const A* __restrict__ gb, int g,
                                       int m1_rt, int n_rt) {
    using O = Op<A, EXACT>;
    m1 = FIXED ? MM1 : m1_rt;
    n = FIXED ? MN : n_rt;
#pragma unroll
    for (int k = 0; k < MM1; ++k) a[k] = (FIXED || k < m1) ? __ldg(ga + (int64_t)g * m1 + k) : A(0);
#pragma unroll
    for (int k = 0; k < NB; ++k)
      b[k] = (MN > 0 && (FIXED || k < n)) ? __ldg(gb + (int64_t)g * n + k) : A(0);
    da[0] = A(0);
#pragma unroll
    for (int k = 1; k < MM1; ++k) da[k - 1] = O::mul(a[k], A(k));
#pragma unroll
    for (int k = 1; k <= NB; ++k) db[k - 1] = O::mul(b[k - 1], A(k));
  }

  __device__ __forceinline__ int dcount() const { return FIXED ? ND : (m1 > 1 ? m1 - 1 : 1); }

  // A(x) = (b_1 + b_2 x + ...) x, 0 when n == 0 (rational.py:211-215)
  __device__ __forceinline__ A series(A x) const {
    using O = Op<A, EXACT>;
    if (MN == 0) return A(0);
    if (!FIXED && n == 0) return A(0);
    return O::mul(horner<A, EXACT, NB, FIXED>(b, n, x), x);
  }

  // y = P(x) / (1 + |A(x)|)  (rational.py:218-224)
  __device__ __forceinline__ A value(A x) const {
    using O = Op<A, EXACT>;
    const A p = horner<A, EXACT, MM1, FIXED>(a, m1, x);
    const A q = O::add(A(1), fabs(series(x)));
    return O::div(p, q);
  }

  // dx, and the m1 + n coefficient-gradient terms folded into acc[]
  // (gradient_terms, rational.py:227-278).
  __device__ __forceinline__ A grad(A x, A u, A (&acc)[KC]) const {
    using O = Op<A, EXACT>;
    const A p = horner<A, EXACT, MM1, FIXED>(a, m1, x);
    const A s = series(x);
    const A q = O::add(A(1), fabs(s));
    const A sg = sign_of(s);
    const A iq = O::rcp(q);
    const A dp = horner<A, EXACT, ND, FIXED>(da, dcount(), x);
    A ds = A(0);
    if (MN > 0 && (FIXED || n > 0)) ds = horner<A, EXACT, NB, FIXED>(db, n, x);
    const A pq = O::mul(p, iq);
    A dx;
    if (EXACT) {
      // u * (dp*iq - ((sg*ds)*pq)*iq), then the da chain t_i = t_{i-1}*x and
      // the db chain from ((-(sg*u))*pq)*iq
      const A t1 = O::mul(dp, iq);
      const A t2 = O::mul(O::mul(O::mul(sg, ds), pq), iq);
      dx = O::mul(u, O::sub(t1, t2));
      A t = O::mul(u, iq);
      acc[0] += t;
#pragma unroll
      for (int i = 1; i < MM1; ++i) {
        t = O::mul(t, x);
        if (FIXED || i < m1) acc[i] += t;
      }
      if (MN > 0 && (FIXED || n > 0)) {
        const A w = O::mul(O::mul(-O::mul(sg, u), pq), iq);
        A v = O::mul(w, x);
        acc[MM1] += v;
#pragma unroll
        for (int j = 1; j < MN; ++j) {
          v = O::mul(v, x);
          if (FIXED || j < n) acc[MM1 + j] += v;
        }
      }
    } else {
      // dx = (u/q) * (P' - sign(A) A' P/q); da_i += (u/q) x^i; db_j += -(sign(A) u/q)(P/q) x^j
      const A t0 = u * iq;
      const A sgds = sg * ds;
      dx = t0 * O::mad(-sgds, pq, dp);
      constexpr int NP = (MM1 - 1 > MN ? MM1 - 1 : MN) + 1;
      A pw[NP];
      pw[0] = A(1);
      if (NP > 1) pw[1] = x;
#pragma unroll
      for (int k = 2; k < NP; ++k) pw[k] = pw[k / 2] * pw[k - k / 2];
      acc[0] += t0;
#pragma unroll
      for (int i = 1; i < MM1; ++i) acc[i] = O::mad(t0, pw[i], acc[i]);
      if (MN > 0) {
        const A w = -(sg * t0) * pq;
#pragma unroll
        for (int j = 0; j < MN; ++j) acc[MM1 + j] = O::mad(w, pw[j + 1], acc[MM1 + j]);
      }
    }
    return dx;
  }
};

}  // namespace grkan
