/*
 * CPU restatement of the SPEC'd Boys kernel, one instantiation per REAL type.
 * Included twice by boys_oracle.c (REAL = double / float).  TEST
 * INFRASTRUCTURE ONLY -- see boys_oracle.c.
 *
 * Follows, operation for operation:
 *   eval_qtilde  SPEC.md:289-297  (Eq. 12: q0 + x (q1 + x q2 u/v), factors in stored order)
 *   eval_fn      SPEC.md:298-306  (t = e^-x; s = Q^n sqrt Q; y = x + s t; r = 1/y;
 *                                  F_n = c r^n sqrt r; x >= z -> r = 1/x, Eq. 4)
 *   binary exponentiation / reciprocal-power form
 *   recursion_fill SPEC.md:307-315 with the index of refmath.py:339-340:
 *                  F_m = (2x F_{m+1} + t) / (2m+1), m = n-1..0, the division
 *                  taken as a multiplication by RN(1/(2m+1))
 *   eval_batch   SPEC.md:316-324  (layouts; domain check of refmath.py:111-115)
 *   eval_with_split SPEC.md:325-333
 */

static REAL SFX(rinv)[64];
static REAL SFX(taylor)[16];

static void SFX(init_consts)(void) {
  for (int m = 0; m < 64; ++m) SFX(rinv)[m] = (REAL)1 / (REAL)(2 * m + 1); /* RN(1/(2m+1)) */
  double f = 1.0;
  for (int k = 0; k < 16; ++k) {       /* RN(1/k!) ; k! exact for k <= 13 (f64), 7 (f32) */
    if (k > 0) f *= k;
    SFX(taylor)[k] = (REAL)1 / (REAL)f;
  }
}

/* e^{-x}, 0 <= x <= XEXP: Cody-Waite with k = round(-x/ln2) via the
 * 1.5*2^(p-1) magic constant, r = -x - k ln2 (hi product exact under FMA),
 * Taylor polynomial of degree TAYLOR_DEG in Horner/FMA form, 2^k scale. */
static REAL SFX(exp_neg)(REAL x) {
  const REAL MAGIC = MAGIC_C;
  REAL kd = FMA(x, -INV_LN2_C, MAGIC);
  REAL kf = kd - MAGIC;
  REAL r = FMA(kf, -LN2_HI_C, -x);
  r = FMA(kf, -LN2_LO_C, r);
  REAL p = SFX(taylor)[TAYLOR_DEG];
  for (int k = TAYLOR_DEG - 1; k >= 0; --k) p = FMA(p, r, SFX(taylor)[k]);
  return p * SFX(pow2)((int)kf);
}

static REAL SFX(exp_neg_clamped)(REAL x) {
  REAL xe = x < XEXP_C ? x : XEXP_C;
  REAL e = SFX(exp_neg)(xe);
  return x <= XEXP_C ? e : (REAL)0;
}

static REAL SFX(powi)(REAL b, int n) { /* n >= 1, LSB first */
  REAL r = b, p = b;
  int have = 0;
  for (int j = 0; (n >> j) != 0; ++j) {
    if ((n >> j) & 1) {
      r = have ? r * p : p;
      have = 1;
    }
    if ((n >> (j + 1)) != 0) p = p * p;
  }
  return r;
}

static REAL SFX(factored)(REAL x, const REAL (*q)[2], int nq, const REAL* l, int nl) {
  REAL acc = 1;
  int first = 1;
  for (int k = 0; k < nq; ++k) {
    REAL d = x - q[k][0];
    REAL f = FMA(d, d, q[k][1]);
    acc = first ? f : acc * f;
    first = 0;
  }
  for (int k = 0; k < nl; ++k) {
    REAL f = x - l[k];
    acc = first ? f : acc * f;
    first = 0;
  }
  return acc;
}

/* eval_qtilde */
static REAL SFX(qtilde)(const SFX(row)* R, REAL x) {
  REAL u = SFX(factored)(x, (const REAL(*)[2])R->uq, R->nuq, R->ul, R->nul);
  REAL v = SFX(factored)(x, (const REAL(*)[2])R->vq, R->nvq, R->vl, R->nvl);
  REAL w = u / v;
  REAL h = R->q2 * w;
  h = FMA(h, x, R->q1);
  return FMA(h, x, R->q0);
}

static int SFX(valid)(REAL x) { return x >= 0 && x <= REAL_MAX_C; }

/* All of F_0..F_n for one x (boys_downward semantics, refmath.py:330-341).
 * Returns 0 and NaNs for x outside the domain. */
static int SFX(point)(const SFX(table)* tb, int n, REAL x, REAL* F, REAL* t_out) {
  if (!SFX(valid)(x)) {
    for (int m = 0; m <= n; ++m) F[m] = (REAL)NAN;
    if (t_out) *t_out = (REAL)NAN;
    return 0;
  }
  const SFX(row)* R = &tb->row[n];
  REAL t = SFX(exp_neg_clamped)(x);
  REAL y = x;
  if (x < R->z) {                                /* eval_fn, below the cut-off */
    REAL Q = SFX(qtilde)(R, x);
    REAL sq = SQRT(Q);
    REAL s = n == 0 ? sq : SFX(powi)(Q, n) * sq;
    y = FMA(s, t, x);
  }
  REAL r = (REAL)1 / y;
  REAL sr = SQRT(r);
  F[n] = n == 0 ? R->c * sr : (R->c * SFX(powi)(r, n)) * sr;
  REAL tx = x + x;
  for (int m = n - 1; m >= 0; --m) F[m] = FMA(tx, F[m + 1], t) * SFX(rinv)[m];
  if (x > R->x_up) {                             /* deep asymptotic: upward ladder */
    REAL rx = (REAL)1 / x;
    REAL f = tb->row[0].c * SQRT(rx);
    F[0] = f;
    for (int m = 0; m < n; ++m) {
      f = (f * ((REAL)m + (REAL)0.5)) * rx;
      F[m + 1] = f;
    }
  }
  if (t_out) *t_out = t;
  return 1;
}
