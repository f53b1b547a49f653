// grkan_math.cuh -- per-element GR-KAN math for sm_100a, two precision policies.
//
// EXACT: the reference's operation order with every *, +, /, 1/q rounded on its
//        own (__fmul_rn / __fadd_rn / __fdiv_rn / __frcp_rn and the packed
//        __fmul2_rn / __fadd2_rn; none is ever contracted into an FMA).  y, dx
//        and each of the m1+n per-element coefficient-gradient terms are then
//        bitwise equal to the reference (pkg/src/grkan/rational.py:195-278;
//        SURVEY.md Appendix A).
// FAST:  FMA Horner, one approximate reciprocal (Q >= 1, so rcp.approx has no
//        denormal corner), powers of x shared by the da and db terms.
//        Restructured but algebraically identical; gated at max-scaled 1e-5.
//
// Two engines:
//   Rational<...>   scalar; any dtype, any degree up to 12/12 (generic path).
//   RationalX2      the hot path: fp32 math at the paper's degrees (5, 4) on
//                   element PAIRS with sm_100a packed FFMA2 / FMUL2 / FADD2,
//                   both policies (EXACT via xmad2's separately rounded steps).
//                   Coefficients stay scalar registers (FFMA2 takes a .F32
//                   broadcast operand), accumulators are float2 pairs.
// Coefficients are CTA-uniform (one group per CTA) and live in registers.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "grkan_types.h"

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

// np.sign for every non-NaN input: +1 / -1, and +0 for both zeros
// (rational.py:251).  A NaN s makes q, 1/q and every output NaN on all paths,
// so the value returned for it is irrelevant.
__device__ __forceinline__ float sign_of(float s) {
  return s == 0.0f ? 0.0f : copysignf(1.0f, s);
}
__device__ __forceinline__ double sign_of(double s) {
  return s == 0.0 ? 0.0 : copysign(1.0, s);
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
// Scalar engine: one coefficient row (one group) in registers.
//   MM1 / MN: compile-time capacity; FIXED: m1 == MM1 and n == MN exactly.
//   Accumulator slot layout: [0, m1) numerator terms, [MM1, MM1 + n) denominator.
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

  // A(x) = (b_1 + b_2 x + ...) x, 0 when n == 0 (rational.py:211-215).
  // ROUNDED: the reference's rounding sequence (needed for sign(A), see grad).
  template <bool ROUNDED = EXACT>
  __device__ __forceinline__ A series(A x) const {
    using O = Op<A, ROUNDED>;
    if (MN == 0) return A(0);
    if (!FIXED && n == 0) return A(0);
    return O::mul(horner<A, ROUNDED, NB, FIXED>(b, n, x), x);
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
    // sign(A) is discontinuous at A's roots: always the reference's rounding.
    const A s = series<true>(x);
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

// ---------------------------------------------------------------------------
// Packed fp32 engine for the paper's degrees (m, n) = (5, 4): element pairs.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float2 bc(float s) { return make_float2(s, s); }  // .F32 broadcast operand
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }

// Separately rounded packed mul + add.  ptxas contracts mul.rn.f32x2 followed
// by add.rn.f32x2 into one FFMA2 (even with explicit .rn), so the add is issued
// as FFMA2(m, one, c) with `one` a kernel parameter the compiler cannot see is
// 1.0: round(m * 1 + c) == round(m + c) exactly (signed zeros included), and the
// product m = round(a * b) must be materialised because it is a multiplicand.
__device__ __forceinline__ float2 xmad2(float2 a, float2 b, float2 c, float one) {
  return fma2(mul2(a, b), bc(one), c);
}
__device__ __forceinline__ float2 xadd2(float2 a, float2 b, float one) { return fma2(a, bc(one), b); }
__device__ __forceinline__ float2 xsub2(float2 a, float2 b, float one) { return fma2(b, bc(-one), a); }

// M1 numerator / N denominator coefficients: the paper's (6, 4) everywhere it is
// the default; (4, 2) for the reference's small test degrees.  Every (6, 4)
// operation sequence is the one the round-1 kernels were verified with.
template <bool EXACT, int M1 = 6, int N = 4>
struct RationalX2 {
  static_assert(M1 >= 3 && M1 <= 6 && N >= 2 && N <= 4, "packed engine degrees");
  static constexpr int KC = M1 + N;
  static constexpr int PMAX = (M1 - 1 > N ? M1 - 1 : N);  // highest power of x in a term
  float a[M1], b[N], da[M1 - 1], db[N];
  float one;  // opaque 1.0 (kernel parameter), see xmad2
  int goff;   // sign-guard scale (FAST): see sign_unsafe

  __device__ __forceinline__ void load(const float* __restrict__ ga, const float* __restrict__ gb, int g,
                                       float one_param) {
    float ab[KC];
#pragma unroll
    for (int k = 0; k < M1; ++k) ab[k] = __ldg(ga + g * M1 + k);
#pragma unroll
    for (int k = 0; k < N; ++k) ab[M1 + k] = __ldg(gb + g * N + k);
    set(ab, one_param);
  }
  // From one row a_0..a_m || b_1..b_n in any memory space (shared-memory tables).
  __device__ __forceinline__ void load_row(const float* ab_row, float one_param) {
    float ab[KC];
#pragma unroll
    for (int k = 0; k < KC; ++k) ab[k] = ab_row[k];
    set(ab, one_param);
  }
  __device__ __forceinline__ void set(const float (&ab)[KC], float one_param) {
#pragma unroll
    for (int k = 0; k < M1; ++k) a[k] = ab[k];
#pragma unroll
    for (int k = 0; k < N; ++k) b[k] = ab[M1 + k];
    da[0] = a[1];  // 1 * a_1 is exact
#pragma unroll
    for (int k = 2; k < M1; ++k) da[k - 1] = __fmul_rn(a[k], float(k));  // fp32 k*a_k, as rational.py:207
    db[0] = b[0];
#pragma unroll
    for (int k = 2; k <= N; ++k) db[k - 1] = __fmul_rn(b[k - 1], float(k));
    one = one_param;
    // sign_unsafe threshold 2^e >= 2^-17 * (|b1| + ... + |bn|), as an exponent
    // offset in float bits; b == 0 (A == 0 exactly) disables it.  Derived for
    // n = 4 (below); for n < 4 the Horner error bound is smaller, so the same
    // threshold is conservative.
    float bsum = fabsf(b[0]);
#pragma unroll
    for (int k = 1; k < N; ++k) bsum += fabsf(b[k]);
    const int eb = static_cast<int>((__float_as_uint(bsum) >> 23) & 0xff) - 126;  // 2^eb > bsum
    goff = bsum > 0.0f ? (eb - 17) * (1 << 23) : -0x7f000000;
  }

  // FAST mode evaluates h = b1 + b2 x + b3 x^2 + b4 x^3 with FMAs, but sign(A)
  // = sign(h x) must be the reference's (sign is discontinuous at A's roots,
  // and a flipped sign moves dx by 2 u A' P / Q^2).  Both Horner forms are
  // within gamma_6 * H(|x|) ~ 3.6e-7 * H of the exact cubic, H(|x|) =
  // sum |b_k| |x|^(k-1) <= bsum * max(1, |x|^3), so their signs can differ
  // only when |h_fma| <= 7.2e-7 * bsum * max(1, |x|^3).  This flags
  // |h| < 2^goff * max(1, |x|^3) (>= 10x margin) with integer compares on the
  // float bits (ALU pipe); flagged pairs recompute h with the reference's
  // separately rounded steps.  Conservative for tiny or huge |h| (wraps to
  // "unsafe").
  // xg = x^(n-1) (x^3 at the paper's degrees).
  __device__ __forceinline__ bool sign_unsafe(float h, float x3) const {
    const float m = fmaxf(fabsf(x3), 1.0f);
    return static_cast<int>((__float_as_uint(h) & 0x7fffffffu) - static_cast<uint32_t>(goff)) <
           static_cast<int>(__float_as_uint(m));
  }

  // -sign(s): -1 / +1 for s > 0 / s < 0, and +0 for s == +-0 (np.sign(0) = 0).
  // One LOP3 (1.0 with the inverted sign bit of s) and one select.
  __device__ __forceinline__ static float neg_sign(float s) {
    const float m = __int_as_float((~__float_as_int(s) & 0x80000000) | 0x3f800000);
    return s == 0.0f ? 0.0f : m;
  }

  // -sign(s) * v without a multiply: flip v's sign bit where s > 0, zero where
  // s == +-0 (np.sign(0) = 0).  One LOP3 and one select.
  __device__ __forceinline__ static float neg_sign_times(float s, float v) {
    const float m = __int_as_float(__float_as_int(v) ^ (~__float_as_int(s) & 0x80000000));
    return s == 0.0f ? 0.0f : m;
  }

  // Horner on a pair with scalar (broadcast) coefficients: the reference's
  // separately rounded acc = acc * x + c (ROUNDED) or FMA steps.
  template <bool ROUNDED, int NC>
  __device__ __forceinline__ float2 horner2(const float (&c)[NC], float2 x) const {
    float2 acc;
    if (ROUNDED) {
      acc = bc(c[NC - 1]);
#pragma unroll
      for (int k = NC - 2; k >= 0; --k) acc = xmad2(acc, x, bc(c[k]), one);
    } else {
      acc = fma2(bc(c[NC - 1]), x, bc(c[NC - 2]));
#pragma unroll
      for (int k = NC - 3; k >= 0; --k) acc = fma2(acc, x, bc(c[k]));
    }
    return acc;
  }

  __device__ __forceinline__ static float rcp(float q) {
    if (EXACT) return __frcp_rn(q);
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(q));
    return r;
  }

  // q = 1 + |A| for a pair: one FADD2 (a single rounding, as the reference's 1.0 + |A|).
  __device__ __forceinline__ static float2 q_of(float2 s) {
    return add2(make_float2(1.0f, 1.0f), make_float2(fabsf(s.x), fabsf(s.y)));
  }

  __device__ __forceinline__ float2 value(float2 x) const {
    const float2 p = horner2<EXACT, M1>(a, x);
    const float2 s = mul2(horner2<EXACT, N>(b, x), x);
    const float2 q = q_of(s);
    if (EXACT) return make_float2(__fdiv_rn(p.x, q.x), __fdiv_rn(p.y, q.y));
    return mul2(p, make_float2(rcp(q.x), rcp(q.y)));
  }

  // FAST: A(x) = h(x) x with h by FMA Horner; `bad` collects sign_unsafe.
  __device__ __forceinline__ float2 series_fast(float2 x, float2 x3, bool& bad) const {
    const float2 h = horner2<false, N>(b, x);
    bad |= sign_unsafe(h.x, x3.x) | sign_unsafe(h.y, x3.y);
    return mul2(h, x);
  }
  // The reference's separately rounded A(x) (EXACT, and FAST's guarded pairs).
  __device__ __forceinline__ float2 series_ref(float2 x) const { return mul2(horner2<true, N>(b, x), x); }

  // dx and the ten coefficient terms of one pair, given A(x) = s.
  // Accumulators: float2 per coefficient (packed FFMA2, the streaming kernels)
  // or one float per coefficient (two scalar FFMAs per pair: the same FMA-pipe
  // cycles, half the registers -- the fused GEMM epilogue).
  static __device__ __forceinline__ void acc_add(float2& a, float2 t) { a = add2(a, t); }
  static __device__ __forceinline__ void acc_add(float& a, float2 t) { a = (a + t.x) + t.y; }
  static __device__ __forceinline__ void acc_fma(float2& a, float2 t, float2 p) { a = fma2(t, p, a); }
  static __device__ __forceinline__ void acc_fma(float& a, float2 t, float2 p) { a = fmaf(t.y, p.y, fmaf(t.x, p.x, a)); }

  // WY: also return the forward value y = P / Q of the pair in *yv (the fused
  // forward + backward step): P/Q rounded once by IEEE division in EXACT mode
  // (rational.py:224, bitwise), P * (1/Q) = pq in FAST mode (K1's FAST form).
  template <bool WY = false, typename ACC>
  __device__ __forceinline__ float2 grad_given(float2 x, float2 u, float2 s, float2 x2, float2 x3,
                                               ACC (&acc)[KC], float2* yv = nullptr) const {
    const float2 p = horner2<EXACT, M1>(a, x);
    const float2 q = q_of(s);
    const float2 iq = make_float2(rcp(q.x), rcp(q.y));
    const float2 dp = horner2<EXACT, M1 - 1>(da, x);
    const float2 ds = horner2<EXACT, N>(db, x);
    const float2 pq = mul2(p, iq);
    if constexpr (WY) *yv = EXACT ? make_float2(__fdiv_rn(p.x, q.x), __fdiv_rn(p.y, q.y)) : pq;
    float2 dx;
    if (EXACT) {
      // dx = u * (dp*iq - ((sg*ds)*pq)*iq); terms t_i = t_{i-1} * x from u*iq;
      // db chain from ((-(sg*u))*pq)*iq -- the reference's order, signed zeros
      // included.  (The accumulations may fuse: only the terms are bitwise.)
      const float2 sg = make_float2(sign_of(s.x), sign_of(s.y));
      const float2 t1 = mul2(dp, iq);
      const float2 t2 = mul2(mul2(mul2(sg, ds), pq), iq);
      dx = mul2(u, xsub2(t1, t2, one));
      float2 t = mul2(u, iq);
      acc_add(acc[0], t);
#pragma unroll
      for (int i = 1; i < M1; ++i) {
        t = mul2(t, x);
        acc_add(acc[i], t);
      }
      float2 v = mul2(mul2(mul2(neg2(mul2(sg, u)), pq), iq), x);
      acc_add(acc[M1], v);
#pragma unroll
      for (int j = 1; j < N; ++j) {
        v = mul2(v, x);
        acc_add(acc[M1 + j], v);
      }
    } else {
      const float2 t0 = mul2(u, iq);
      // z = -sign(A) P/q on the ALU pipe (sign flip + select), not the FMA pipe
      const float2 z = make_float2(neg_sign_times(s.x, pq.x), neg_sign_times(s.y, pq.y));
      dx = mul2(t0, fma2(ds, z, dp));               // (u/q) (P' - sign(A) A' P/q)
      const float2 w = mul2(t0, z);                 // -(sign(A) u/q) P/q
      float2 pw[PMAX + 1];                          // x^1..x^PMAX: x^4 = x^2 x^2, x^5 = x^4 x
      pw[1] = x;
      pw[2] = x2;
      if constexpr (PMAX >= 3) pw[3] = x3;
      if constexpr (PMAX >= 4) pw[4] = mul2(x2, x2);
      if constexpr (PMAX >= 5) pw[5] = mul2(pw[4], x);
      acc_add(acc[0], t0);
#pragma unroll
      for (int i = 1; i < M1; ++i) acc_fma(acc[i], t0, pw[i]);
#pragma unroll
      for (int j = 0; j < N; ++j) acc_fma(acc[M1 + j], w, pw[j + 1]);
    }
    return dx;
  }

  // ---- bf16 I/O, FAST: the x-only factors from a per-CTA table ----------------
  // A bf16 x takes at most 2^16 values, and of the per-element quantities only
  // u enters linearly: t0 = u * (1/Q) and w = u * (-sign(A) P / Q^2).  So each
  // CTA tabulates {1/Q, -sign(A) P/Q^2} over a window of x exponents once, and
  // the streaming body keeps only what involves u or the powers of x.
  // lut_entry is the one definition of a table entry (also the out-of-window
  // fallback, so an element's result never depends on which served it): A with
  // the reference's separately rounded steps (exact sign(A), rational.py:211-215,
  // 251), P by FMA Horner, 1/Q by IEEE reciprocal.
  __device__ __forceinline__ float2 lut_entry(float x) const {
    static_assert(M1 == 6 && N == 4, "the bf16 table body is written for the paper's degrees");
    float h = b[3];
#pragma unroll
    for (int k = 2; k >= 0; --k) h = __fadd_rn(__fmul_rn(h, x), b[k]);
    const float s = __fmul_rn(h, x);
    float p = fmaf(a[5], x, a[4]);
#pragma unroll
    for (int k = 3; k >= 0; --k) p = fmaf(p, x, a[k]);
    const float iq = __frcp_rn(__fadd_rn(1.0f, fabsf(s)));
    const float z = neg_sign_times(s, p * iq);  // -sign(A) P/Q
    return make_float2(iq, iq * z);
  }

  // dx and the ten terms of one pair given its table entries iq = 1/Q and
  // wq = -sign(A)P/Q^2: 25 packed FP32 ops per pair instead of grad_given's 39, no MUFU.
  template <typename ACC>
  __device__ __forceinline__ float2 grad_lut(float2 x, float2 u, float2 iq, float2 wq, ACC (&acc)[KC]) const {
    static_assert(M1 == 6 && N == 4, "the bf16 table body is written for the paper's degrees");
    const float2 t0 = mul2(u, iq);  // u/Q
    const float2 w = mul2(u, wq);   // -sign(A) u P/Q^2
    const float2 dp = horner2<false, 5>(da, x);
    const float2 ds = horner2<false, 4>(db, x);
    const float2 dx = fma2(w, ds, mul2(t0, dp));         // u (P'/Q - sign(A) A' P/Q^2)
    const float2 x2 = mul2(x, x);
    const float2 x3 = mul2(x2, x);
    const float2 x4 = mul2(x2, x2);
    const float2 x5 = mul2(x4, x);
    acc_add(acc[0], t0);
    acc_fma(acc[1], t0, x);
    acc_fma(acc[2], t0, x2);
    acc_fma(acc[3], t0, x3);
    acc_fma(acc[4], t0, x4);
    acc_fma(acc[5], t0, x5);
    acc_fma(acc[6], w, x);
    acc_fma(acc[7], w, x2);
    acc_fma(acc[8], w, x3);
    acc_fma(acc[9], w, x4);
    return dx;
  }

  // dx for NP pairs (one 16-byte vector) and their terms folded into acc.
  // FAST: the guard is evaluated for all NP pairs first and resolved by ONE
  // (rarely taken) branch, so the straight-line math of the NP pairs stays in
  // one basic block the scheduler can interleave.
  // GRKAN_GUARD_NP pairs share one guard branch (tuning knob; the pairs'
  // x^2 / x^3 stay live across it).  GUARD = false evaluates A(x) with the
  // reference's rounding in FAST mode too: measured faster for bf16 I/O, whose
  // backward is latency-bound and loses more to the guard's branches than it
  // gains from 3 fewer FMUL2 per pair (fp32: 323 -> 307 us with the guard,
  // bf16: 260 -> 273 us at KAT-B; 283 us with a warp-uniform __any_sync branch).
  template <int NP, bool GUARD = true, typename ACC = float2, bool WY = false>
  __device__ __forceinline__ void grad_n(const float (&vx)[2 * NP], const float (&vu)[2 * NP],
                                         float (&o)[2 * NP], ACC (&acc)[KC],
                                         float (*yo)[2 * NP] = nullptr) const {
    constexpr int G = GRKAN_GUARD_NP < NP ? GRKAN_GUARD_NP : NP;
    static_assert(NP % G == 0, "guard group must divide the pair count");
#pragma unroll
    for (int i0 = 0; i0 < NP; i0 += G) {
      float2 x[G], s[G], x2[G], x3[G];
#pragma unroll
      for (int i = 0; i < G; ++i) x[i] = make_float2(vx[2 * (i0 + i)], vx[2 * (i0 + i) + 1]);
      if (EXACT || !GUARD || !GRKAN_SIGN_GUARD) {
#pragma unroll
        for (int i = 0; i < G; ++i) {
          s[i] = series_ref(x[i]);
          if (!EXACT) {
            x2[i] = mul2(x[i], x[i]);
            x3[i] = mul2(x2[i], x[i]);
          }
        }
      } else {
        bool bad = false;
#pragma unroll
        for (int i = 0; i < G; ++i) {
          x2[i] = mul2(x[i], x[i]);
          x3[i] = mul2(x2[i], x[i]);
          s[i] = series_fast(x[i], x3[i], bad);
        }
        if (bad) {
#pragma unroll
          for (int i = 0; i < G; ++i) s[i] = series_ref(x[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < G; ++i) {
        const int e = 2 * (i0 + i);
        float2 yv;
        const float2 r = grad_given<WY>(x[i], make_float2(vu[e], vu[e + 1]), s[i], x2[i], x3[i], acc, &yv);
        o[e] = r.x;
        o[e + 1] = r.y;
        if constexpr (WY) {
          (*yo)[e] = yv.x;
          (*yo)[e + 1] = yv.y;
        }
      }
    }
  }
};

}  // namespace grkan
