/*
 * boys_quad -- extended-precision restatements of the reference ORACLE
 * (refmath.boys_downward), for accuracy scans at the paper's density
 * (~2^20 points per order), where the mpmath oracle
 * (~1 ms per point) is too slow.
 *
 * TEST INFRASTRUCTURE, NOT PRODUCT CODE (only tests/ load it).
 *
 * Two instantiations of one algorithm:
 *   boys_quad_downward : binary128 (libquadmath), ~2^-106 (slow: ~0.4 ms/pt)
 *   boys_ld_downward   : x87 80-bit long double, ~2^-60 (fast: a few us/pt)
 * Algorithms follow refmath.py at the working precision:
 *   x == 0        -> 1/(2n+1)                                   refmath.py:300-301
 *   x <  n + 20   -> power series with geometric tail stop       refmath.py:134-157
 *   x >= n + 20   -> Legendre continued fraction for the upper
 *                    incomplete gamma, modified Lentz             refmath.py:205-248
 *   all orders    -> F_n seed + downward recursion
 *                    F_m = (2x F_{m+1} + e^-x)/(2m+1)            refmath.py:330-341
 * Output: double-double (hi, lo) per value, [N][n+1][2].  Pinned against the
 * mpmath goldens in tests/test_quad_reference.py.
 */
#include <math.h>
#include <quadmath.h>
#include <stdint.h>

/* glibc's x87 expl/powl serialise across threads; these are plain
 * arithmetic (reduction by ln2 in two parts + Taylor to 2^-66). */
static long double exp_ld(long double x) {
  const long double LN2_HI = 0.693147180559945309417232121458176568L;
  const long double LN2_LO = 1.0e-40L * 0;   /* LN2_HI is RN64(ln 2); residue < 2^-65 */
  long double k = (long double)(long long)(x / LN2_HI + 0.5L);   /* x >= 0 here; nearbyintl is slow */
  long double r = (x - k * LN2_HI) - k * LN2_LO;
  long double t = 1, s = 1;
  for (int i = 1; i < 24; ++i) {
    t *= r / i;
    s += t;
  }
  return ldexpl(s, (int)k);
}
static long double pow_ld(long double x, long double a) { /* x^a, a = -(n + 1/2) */
  int n = (int)(-a - 0.5L);
  long double p = 1;
  for (int k = 0; k < n; ++k) p *= x;
  return 1 / (p * sqrtl(x));
}

#define DEFINE_BOYS(R, SFX, EXP, POW, SQRT, FABS, PI, TOL, EPS, TINY)                     \
  static R cn_##SFX(int n) { /* c_n = Gamma(n+1/2)/2 */                                    \
    R c = SQRT(PI) / 2;                                                                    \
    for (int k = 1; k <= n; ++k) c *= (R)(2 * k - 1) / 2;                                  \
    return c;                                                                              \
  }                                                                                        \
  static R series_##SFX(int n, R x) {                                                      \
    R twox = 2 * x, term = (R)1 / (2 * n + 1), total = term;                               \
    for (long k = 1; k < 4000000; ++k) {                                                   \
      term *= twox / (2 * n + 2 * k + 1);                                                  \
      total += term;                                                                       \
      R d = 2 * n + 2 * k + 3;                                                             \
      /* geometric tail bound term*r/(1-r) < tol*total with r = 2x/d, division-free */     \
      if (twox < d && term * twox < TOL * total * (d - twox)) break;                       \
    }                                                                                      \
    return EXP(-x) * total;                                                                \
  }                                                                                        \
  static R upper_cf_##SFX(int n, R x) {                                                    \
    const R a = (R)(2 * n + 1) / 2;                                                        \
    R b0 = x + 1 - a;                                                                      \
    R f = b0 != 0 ? b0 : TINY, C = f, D = 0;                                               \
    int hits = 0;                                                                          \
    for (long j = 1; j < 100000; ++j) {                                                    \
      R am = j * (a - j), bm = x + 2 * j + 1 - a;                                          \
      D = bm + am * D;                                                                     \
      if (D == 0) D = TINY;                                                                \
      C = bm + am / C;                                                                     \
      if (C == 0) C = TINY;                                                                \
      D = 1 / D;                                                                           \
      R delta = C * D;                                                                     \
      f *= delta;                                                                          \
      if (FABS(delta - 1) < EPS) {                                                         \
        if (++hits >= 2) break;                                                            \
      } else {                                                                             \
        hits = 0;                                                                          \
      }                                                                                    \
    }                                                                                      \
    /* (Gamma(a) - e^-x x^a / f) / (2 x^a), arranged so x^a cannot overflow */             \
    return cn_##SFX(n) * POW(x, -a) - EXP(-x) / (2 * f);                                   \
  }                                                                                        \
  static R boys_##SFX(int n, R x) {                                                        \
    if (x == 0) return (R)1 / (2 * n + 1);                                                 \
    if (x < n + 20) return series_##SFX(n, x);                                             \
    return upper_cf_##SFX(n, x);                                                           \
  }                                                                                        \
  void boys_##SFX##_downward(int n, const double* x, int64_t N, double* out) {             \
    _Pragma("omp parallel for schedule(dynamic, 256)")                                     \
    for (int64_t i = 0; i < N; ++i) {                                                      \
      R xq = x[i];                                                                         \
      R F[130];                                                                            \
      F[n] = boys_##SFX(n, xq);                                                            \
      R ex = EXP(-xq);                                                                     \
      for (int m = n - 1; m >= 0; --m) F[m] = (2 * xq * F[m + 1] + ex) / (2 * m + 1);      \
      for (int m = 0; m <= n; ++m) {                                                       \
        double hi = (double)F[m];                                                          \
        double lo = (double)(F[m] - (R)hi);                                                \
        out[(i * (n + 1) + m) * 2] = hi;                                                   \
        out[(i * (n + 1) + m) * 2 + 1] = lo;                                               \
      }                                                                                    \
    }                                                                                      \
  }

DEFINE_BOYS(__float128, quad, expq, powq, sqrtq, fabsq, M_PIq, 0x1p-112Q, 0x1p-111Q, 0x1p-16000Q)
DEFINE_BOYS(long double, ld, exp_ld, pow_ld, sqrtl, fabsl, 3.14159265358979323846264338327950288L,
            0x1p-63L, 0x1p-62L, 0x1p-16000L)
