/*
 * Precision-generic body of the C oracle -- TEST INFRASTRUCTURE ONLY.
 * Included twice by grkan_oracle.c with REAL = float / double and SUF = f / d.
 * See grkan_oracle.c for the reference citations.
 */
#define CAT2(a, b) a##_##b
#define CAT(a, b) CAT2(a, b)
#define FN(name) CAT(name, SUF)

typedef struct {
  REAL a[MAXC], b[MAXC], da[MAXC], db[MAXC];
  int m1, n;
} FN(coef);

/* coefficients cast to the run dtype at use (rational.py:220-221, 243-244);
 * derivative coefficients k*c_k in the run dtype (rational.py:203-208, 255) */
static void FN(coef_init)(FN(coef) * c, const double* num, const double* den, int m1, int n) {
  c->m1 = m1;
  c->n = n;
  for (int k = 0; k < m1; ++k) c->a[k] = (REAL)num[k];
  for (int k = 0; k < n; ++k) c->b[k] = (REAL)den[k];
  c->da[0] = (REAL)0;
  for (int k = 1; k < m1; ++k) c->da[k - 1] = c->a[k] * (REAL)k;
  for (int k = 1; k <= n; ++k) c->db[k - 1] = c->b[k - 1] * (REAL)k;
}

/* Horner, top coefficient first, separately rounded (rational.py:195-200) */
static inline REAL FN(horner)(const REAL* c, int cnt, REAL x) {
  REAL acc = c[cnt - 1];
  for (int k = cnt - 2; k >= 0; --k) {
    acc = acc * x;
    acc = acc + c[k];
  }
  return acc;
}

/* P(x) / (1 + |A(x)|) (rational.py:218-224) */
static inline REAL FN(value)(const FN(coef) * c, REAL x) {
  REAL p = FN(horner)(c->a, c->m1, x);
  REAL s = c->n ? FN(horner)(c->b, c->n, x) * x : (REAL)0;
  REAL q = (REAL)1 + (REAL)fabs((double)s);
  return p / q;
}

/* gradient_terms (rational.py:227-278): returns dx, fills ta[m1], tb[n] */
static inline REAL FN(terms)(const FN(coef) * c, REAL x, REAL u, REAL* ta, REAL* tb) {
  REAL p = FN(horner)(c->a, c->m1, x);
  REAL s = c->n ? FN(horner)(c->b, c->n, x) * x : (REAL)0;
  REAL q = (REAL)1 + (REAL)fabs((double)s);
  REAL sg = s > (REAL)0 ? (REAL)1 : (s < (REAL)0 ? (REAL)-1 : (s == (REAL)0 ? (REAL)0 : s));
  REAL iq = (REAL)1 / q;
  REAL dp = FN(horner)(c->da, c->m1 > 1 ? c->m1 - 1 : 1, x);
  REAL ds = c->n ? FN(horner)(c->db, c->n, x) : (REAL)0;
  REAL pq = p * iq;
  REAL t1 = dp * iq;
  REAL t2 = sg * ds;
  t2 = t2 * pq;
  t2 = t2 * iq;
  REAL dx = u * (t1 - t2);
  REAL t = u * iq;
  ta[0] = t;
  for (int i = 1; i < c->m1; ++i) {
    t = t * x;
    ta[i] = t;
  }
  if (c->n) {
    REAL w = -(sg * u);
    w = w * pq;
    w = w * iq;
    REAL v = w * x;
    tb[0] = v;
    for (int j = 1; j < c->n; ++j) {
      v = v * x;
      tb[j] = v;
    }
  }
  return dx;
}

/* forward_tensor (rational.py:325-345) */
void FN(orc_fwd)(const REAL* x, REAL* y, const double* num, const double* den, int64_t rows,
                 int32_t d, int32_t ng, int32_t m1, int32_t n) {
  int32_t dg = d / ng;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r) {
    for (int32_t g = 0; g < ng; ++g) {
      FN(coef) c;
      FN(coef_init)(&c, num + (int64_t)g * m1, den + (int64_t)g * n, m1, n);
      const REAL* xr = x + r * d + (int64_t)g * dg;
      REAL* yr = y + r * d + (int64_t)g * dg;
      for (int32_t f = 0; f < dg; ++f) yr[f] = FN(value)(&c, xr[f]);
    }
  }
}

/*
 * All backward products in one pass per group.  OpenMP runs groups in parallel;
 * every fold is sequential inside one thread, so results do not depend on the
 * thread count.  Any output pointer may be NULL.
 *   blk_*  backward_blocked, tensor dtype (backward.py:122-139 then ordered
 *          combine from zero, :142-179)
 *   nav_*  backward_naive, tensor dtype (backward.py:113-119, 226-229)
 *   ref_*  reference_coeff_grads: double fold of the run-dtype terms
 *          (verification.py:318-341)
 *   tru_*  terms evaluated in double from the run-dtype inputs/coefficients,
 *          Neumaier-compensated double fold (the "true fp64" oracle)
 * Returns 1 when a blocked or naive accumulator is non-finite
 * (_check_accumulators, backward.py:182-184).
 */
int FN(orc_bwd)(const REAL* x, const REAL* u, const double* num, const double* den,
                int64_t rows, int32_t d, int32_t ng, int32_t m1, int32_t n, int64_t block,
                REAL* dx, REAL* blk_da, REAL* blk_db, REAL* nav_da, REAL* nav_db,
                double* ref_da, double* ref_db, double* tru_da, double* tru_db) {
  int32_t dg = d / ng;
  int bad = 0;
  int want_true = tru_da != 0 || tru_db != 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
  for (int32_t g = 0; g < ng; ++g) {
    FN(coef) c;
    FN(coef_init)(&c, num + (int64_t)g * m1, den + (int64_t)g * n, m1, n);
    coef_dbl cd;
    {
      double nr[MAXC], dr[MAXC];
      for (int k = 0; k < m1; ++k) nr[k] = (double)c.a[k];
      for (int k = 0; k < n; ++k) dr[k] = (double)c.b[k];
      coef_init_dbl(&cd, nr, dr, m1, n);
    }
    REAL ta[MAXC], tb[MAXC], pa[MAXC], pb[MAXC], ga[MAXC], gb[MAXC], sa[MAXC], sb[MAXC];
    double ra[MAXC], rb[MAXC], ea[MAXC], eb[MAXC], ca[MAXC], cb[MAXC], ta64[MAXC], tb64[MAXC];
    for (int k = 0; k < MAXC; ++k) {
      ga[k] = gb[k] = sa[k] = sb[k] = (REAL)0;
      ra[k] = rb[k] = ea[k] = eb[k] = ca[k] = cb[k] = 0.0;
    }
    int64_t seen = 0;
    for (int64_t r0 = 0; r0 < rows; r0 += block) {
      int64_t r1 = r0 + block < rows ? r0 + block : rows;
      int64_t inblk = 0;
      for (int64_t r = r0; r < r1; ++r) {
        for (int32_t f = 0; f < dg; ++f) {
          int64_t e = r * d + (int64_t)g * dg + f;
          REAL dxe = FN(terms)(&c, x[e], u[e], ta, tb);
          if (dx) dx[e] = dxe;
          /* np.add.accumulate starts from the first element, not from zero */
          for (int i = 0; i < m1; ++i) {
            pa[i] = inblk ? pa[i] + ta[i] : ta[i];
            sa[i] = seen ? sa[i] + ta[i] : ta[i];
            ra[i] = seen ? ra[i] + (double)ta[i] : (double)ta[i];
          }
          for (int j = 0; j < n; ++j) {
            pb[j] = inblk ? pb[j] + tb[j] : tb[j];
            sb[j] = seen ? sb[j] + tb[j] : tb[j];
            rb[j] = seen ? rb[j] + (double)tb[j] : (double)tb[j];
          }
          if (want_true) {
            terms_dbl(&cd, (double)x[e], (double)u[e], ta64, tb64);
            for (int i = 0; i < m1; ++i) {
              double t0 = ea[i] + ta64[i];
              ca[i] += fabs(ea[i]) >= fabs(ta64[i]) ? (ea[i] - t0) + ta64[i] : (ta64[i] - t0) + ea[i];
              ea[i] = t0;
            }
            for (int j = 0; j < n; ++j) {
              double t0 = eb[j] + tb64[j];
              cb[j] += fabs(eb[j]) >= fabs(tb64[j]) ? (eb[j] - t0) + tb64[j] : (tb64[j] - t0) + eb[j];
              eb[j] = t0;
            }
          }
          ++inblk;
          ++seen;
        }
      }
      if (inblk) { /* ordered combine from zeros, ascending row-block */
        for (int i = 0; i < m1; ++i) ga[i] = ga[i] + pa[i];
        for (int j = 0; j < n; ++j) gb[j] = gb[j] + pb[j];
      }
    }
    for (int i = 0; i < m1; ++i) {
      int64_t o = (int64_t)g * m1 + i;
      if (blk_da) blk_da[o] = ga[i];
      if (nav_da) nav_da[o] = sa[i];
      if (ref_da) ref_da[o] = ra[i];
      if (tru_da) tru_da[o] = ea[i] + ca[i];
      if (!isfinite((double)ga[i]) || !isfinite((double)sa[i])) bad |= 1;
    }
    for (int j = 0; j < n; ++j) {
      int64_t o = (int64_t)g * n + j;
      if (blk_db) blk_db[o] = gb[j];
      if (nav_db) nav_db[o] = sb[j];
      if (ref_db) ref_db[o] = rb[j];
      if (tru_db) tru_db[o] = eb[j] + cb[j];
      if (!isfinite((double)gb[j]) || !isfinite((double)sb[j])) bad |= 1;
    }
  }
  return bad;
}

#undef FN
#undef CAT
#undef CAT2
