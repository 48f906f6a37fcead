/*
 * boys_oracle -- CPU restatement of the batched Boys evaluator.
 *
 * TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke()
 * and bench.py's CPU-baseline leg may load this library, and only as the
 * checker (or the timed CPU reference arm); the product path (libboys.so)
 * never calls it and has no CPU fallback.
 *
 * What it restates: the reference ships the Boys kernel only as a
 * specification plus the arbitrary-precision template
 * boys_downward (refmath.py:330-341).  This file implements that kernel in
 * plain C99 with explicit fma(), IEEE division and sqrt, no contraction
 * (-ffp-contract=off), and its own table loader: it parses the hex-float
 * dataset (paper_2504_07637_b200/data/boys_*.dat) directly, so it shares no
 * code with the CUDA path -- not even the generated header.
 *
 * Pinning: tests/test_oracle.py checks it against golden vectors computed
 * from the reference oracle refmath.boys_downward at Precision(96)
 * (tests/golden/make_golden.py) to the paper's Table I bounds, and against
 * the SPEC's known-answer examples.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define MAXQ 8
#define MAXL 2
#define MAXN 64

/* ---------------- f64 instantiation ---------------- */
typedef struct {
  double q0, q1, q2, c, z, x_up;
  double uq[MAXQ][2], ul[MAXL], vq[MAXQ][2], vl[MAXL];
  int nuq, nul, nvq, nvl, N;
} row_f64;
typedef struct {
  int max_order;
  row_f64 row[MAXN];
} table_f64;

static double pow2_f64(int k) { /* 2^k, normal range */
  uint64_t b = (uint64_t)(k + 1023) << 52;
  double d;
  memcpy(&d, &b, 8);
  return d;
}

#define REAL double
#define SFX(name) name##_f64
#define FMA fma
#define SQRT sqrt
#define MAGIC_C 0x1.8p52
#define INV_LN2_C 0x1.71547652b82fep+0
#define LN2_HI_C 0x1.62e42fefa39efp-1   /* RN(ln 2) */
#define LN2_LO_C 0x1.abc9e3b39803fp-56  /* RN(ln 2 - LN2_HI) */
#define TAYLOR_DEG 13
#define XEXP_C 708.0
#define REAL_MAX_C 0x1.fffffffffffffp+1023
#include "boys_oracle_impl.h"
#undef REAL
#undef SFX
#undef FMA
#undef SQRT
#undef MAGIC_C
#undef INV_LN2_C
#undef LN2_HI_C
#undef LN2_LO_C
#undef TAYLOR_DEG
#undef XEXP_C
#undef REAL_MAX_C

/* ---------------- f32 instantiation ---------------- */
typedef struct {
  float q0, q1, q2, c, z, x_up;
  float uq[MAXQ][2], ul[MAXL], vq[MAXQ][2], vl[MAXL];
  int nuq, nul, nvq, nvl, N;
} row_f32;
typedef struct {
  int max_order;
  row_f32 row[MAXN];
} table_f32;

static float pow2_f32(int k) {
  uint32_t b = (uint32_t)(k + 127) << 23;
  float f;
  memcpy(&f, &b, 4);
  return f;
}

#define REAL float
#define SFX(name) name##_f32
#define FMA fmaf
#define SQRT sqrtf
#define MAGIC_C 0x1.8p23f
#define INV_LN2_C 0x1.715476p+0f
#define LN2_HI_C 0x1.62e430p-1f        /* RN32(ln 2) */
#define LN2_LO_C -0x1.05c610p-29f      /* RN32(ln 2 - LN2_HI) */
#define TAYLOR_DEG 7
#define XEXP_C 86.0f
#define REAL_MAX_C 0x1.fffffep+127f
#include "boys_oracle_impl.h"

/* ---------------- dataset loader (coeffs file format) ---- */

typedef struct {
  int is_f32;
  table_f64 t64;
  table_f32 t32;
} oracle_table;

static int next_tok(FILE* f, char* buf, size_t cap) {
  int c;
  for (;;) {
    c = fgetc(f);
    if (c == EOF) return 0;
    if (c == '#') {
      while (c != '\n' && c != EOF) c = fgetc(f);
      continue;
    }
    if (c > ' ') break;
  }
  size_t k = 0;
  while (c != EOF && c > ' ') {
    if (k + 1 < cap) buf[k++] = (char)c;
    c = fgetc(f);
  }
  buf[k] = 0;
  return 1;
}

static int expect(FILE* f, const char* key) {
  char b[128];
  return next_tok(f, b, sizeof b) && strcmp(b, key) == 0;
}
static int read_int(FILE* f, int* v) {
  char b[128];
  if (!next_tok(f, b, sizeof b)) return 0;
  *v = atoi(b);
  return 1;
}
static int read_real(FILE* f, double* v) {
  char b[128];
  if (!next_tok(f, b, sizeof b)) return 0;
  char* end;
  *v = strtod(b, &end); /* hex floats parse exactly */
  return *end == 0;
}

/* Returns NULL on any parse error.  (Checksum verification is done by the
 * Python loader; this parser only needs the values.) */
void* boys_oracle_load(const char* path) {
  FILE* f = fopen(path, "r");
  if (!f) return NULL;
  oracle_table* ot = calloc(1, sizeof *ot);
  char b[128];
  int ver, cnt, ok = 1;
  ok = ok && expect(f, "version") && read_int(f, &ver) && ver == 1;
  ok = ok && expect(f, "profile") && next_tok(f, b, sizeof b);
  if (ok) ot->is_f32 = strcmp(b, "single24") == 0;
  ok = ok && expect(f, "orders") && read_int(f, &cnt) && cnt > 0 && cnt <= MAXN;
  for (int r = 0; ok && r < cnt; ++r) {
    int n, N;
    ok = expect(f, "record") && read_int(f, &n) && read_int(f, &N) && n == r;
    double sc[8];
    const char* names[8] = {"c", "q0", "q1", "q2", "alpha", "beta", "z", "x_up"};
    for (int k = 0; ok && k < 8; ++k) ok = expect(f, names[k]) && read_real(f, &sc[k]);
    double eb;
    ok = ok && expect(f, "exact_bits") && read_real(f, &eb);
    double uq[MAXQ][2] = {{0}}, vq[MAXQ][2] = {{0}}, ul[MAXL] = {0}, vl[MAXL] = {0};
    int nuq = 0, nul = 0, nvq = 0, nvl = 0;
    ok = ok && expect(f, "u_quads") && read_int(f, &nuq) && nuq <= MAXQ;
    for (int k = 0; ok && k < nuq; ++k) ok = read_real(f, &uq[k][0]) && read_real(f, &uq[k][1]);
    ok = ok && expect(f, "u_lins") && read_int(f, &nul) && nul <= MAXL;
    for (int k = 0; ok && k < nul; ++k) ok = read_real(f, &ul[k]);
    ok = ok && expect(f, "v_quads") && read_int(f, &nvq) && nvq <= MAXQ;
    for (int k = 0; ok && k < nvq; ++k) ok = read_real(f, &vq[k][0]) && read_real(f, &vq[k][1]);
    ok = ok && expect(f, "v_lins") && read_int(f, &nvl) && nvl <= MAXL;
    for (int k = 0; ok && k < nvl; ++k) ok = read_real(f, &vl[k]);
    ok = ok && expect(f, "end");
    if (!ok) break;
#define FILL(RW, T)                                                           \
  do {                                                                        \
    RW->c = (T)sc[0]; RW->q0 = (T)sc[1]; RW->q1 = (T)sc[2]; RW->q2 = (T)sc[3]; \
    RW->z = (T)sc[6]; RW->x_up = (T)sc[7];                                    \
    RW->nuq = nuq; RW->nul = nul; RW->nvq = nvq; RW->nvl = nvl; RW->N = N;    \
    for (int k = 0; k < MAXQ; ++k) {                                          \
      RW->uq[k][0] = (T)uq[k][0]; RW->uq[k][1] = (T)uq[k][1];                 \
      RW->vq[k][0] = (T)vq[k][0]; RW->vq[k][1] = (T)vq[k][1];                 \
    }                                                                         \
    for (int k = 0; k < MAXL; ++k) { RW->ul[k] = (T)ul[k]; RW->vl[k] = (T)vl[k]; } \
  } while (0)
    if (ot->is_f32) {
      row_f32* rw = &ot->t32.row[n];
      FILL(rw, float);
      ot->t32.max_order = n;
    } else {
      row_f64* rw = &ot->t64.row[n];
      FILL(rw, double);
      ot->t64.max_order = n;
    }
  }
  fclose(f);
  if (!ok) {
    free(ot);
    return NULL;
  }
  init_consts_f64();
  init_consts_f32();
  return ot;
}

void boys_oracle_free(void* t) { free(t); }

int boys_oracle_max_order(const void* t) {
  const oracle_table* ot = t;
  return ot->is_f32 ? ot->t32.max_order : ot->t64.max_order;
}
int boys_oracle_is_f32(const void* t) { return ((const oracle_table*)t)->is_f32; }

/* Dense batch: layout 0 = SoA [n+1][N], 1 = AoS [N][n+1].  expx nullable.
 * Returns the first offending index, or -1 when every x is in the domain. */
int64_t boys_oracle_dense(const void* t, int n, const void* x, int64_t N, void* out, int layout,
                          void* expx) {
  const oracle_table* ot = t;
  const int W = n + 1;
  int64_t first_bad = INT64_MAX;
#pragma omp parallel for schedule(static) reduction(min : first_bad)
  for (int64_t i = 0; i < N; ++i) {
    int ok;
    if (ot->is_f32) {
      float F[MAXN + 1], tt;
      ok = point_f32(&ot->t32, n, ((const float*)x)[i], F, &tt);
      for (int m = 0; m < W; ++m)
        ((float*)out)[layout ? i * W + m : (int64_t)m * N + i] = F[m];
      if (expx) ((float*)expx)[i] = tt;
    } else {
      double F[MAXN + 1], tt;
      ok = point_f64(&ot->t64, n, ((const double*)x)[i], F, &tt);
      for (int m = 0; m < W; ++m)
        ((double*)out)[layout ? i * W + m : (int64_t)m * N + i] = F[m];
      if (expx) ((double*)expx)[i] = tt;
    }
    if (!ok && i < first_bad) first_bad = i;
  }
  return first_bad == INT64_MAX ? -1 : first_bad;
}

/* Ragged batch: element i of order nmax[i] at out[offsets[i] + m]. */
int64_t boys_oracle_ragged(const void* t, const void* x, const uint8_t* nmax,
                           const int64_t* offsets, int64_t N, void* out) {
  const oracle_table* ot = t;
  int64_t first_bad = INT64_MAX;
#pragma omp parallel for schedule(static) reduction(min : first_bad)
  for (int64_t i = 0; i < N; ++i) {
    int n = nmax[i], ok;
    if (n > boys_oracle_max_order(t)) {
      ok = 0;
      for (int m = 0; m <= n; ++m) {
        if (ot->is_f32) ((float*)out)[offsets[i] + m] = NAN;
        else ((double*)out)[offsets[i] + m] = NAN;
      }
    } else if (ot->is_f32) {
      ok = point_f32(&ot->t32, n, ((const float*)x)[i], (float*)out + offsets[i], NULL);
    } else {
      ok = point_f64(&ot->t64, n, ((const double*)x)[i], (double*)out + offsets[i], NULL);
    }
    if (!ok && i < first_bad) first_bad = i;
  }
  return first_bad == INT64_MAX ? -1 : first_bad;
}

/* eval_with_split: F_0..F_nbar from the order-nbar seed,
 * F_{nbar+1}..F_n from the order-n seed. */
int64_t boys_oracle_split(const void* t, int n, int nbar, const void* x, int64_t N, void* out,
                          int layout) {
  const oracle_table* ot = t;
  const int W = n + 1;
  int64_t first_bad = INT64_MAX;
#pragma omp parallel for schedule(static) reduction(min : first_bad)
  for (int64_t i = 0; i < N; ++i) {
    int ok;
    if (ot->is_f32) {
      float Fh[MAXN + 1], Fl[MAXN + 1];
      ok = point_f32(&ot->t32, n, ((const float*)x)[i], Fh, NULL);
      point_f32(&ot->t32, nbar, ((const float*)x)[i], Fl, NULL);
      for (int m = 0; m < W; ++m)
        ((float*)out)[layout ? i * W + m : (int64_t)m * N + i] = m <= nbar ? Fl[m] : Fh[m];
    } else {
      double Fh[MAXN + 1], Fl[MAXN + 1];
      ok = point_f64(&ot->t64, n, ((const double*)x)[i], Fh, NULL);
      point_f64(&ot->t64, nbar, ((const double*)x)[i], Fl, NULL);
      for (int m = 0; m < W; ++m)
        ((double*)out)[layout ? i * W + m : (int64_t)m * N + i] = m <= nbar ? Fl[m] : Fh[m];
    }
    if (!ok && i < first_bad) first_bad = i;
  }
  return first_bad == INT64_MAX ? -1 : first_bad;
}

/* Fused consumer: McMurchie-Davidson Hermite Coulomb
 * integrals pref * R^{(0)}_{tuv}, t+u+v <= L, for every (bra pair i, ket pair
 * j); pair records are 5 doubles (p, Px, Py, Pz, K).  The operation sequence
 * of csrc/hermite.cu (Helgaker's recurrences, in place, level n = L-1..0 in
 * decreasing order s = t+u+v), in C with explicit fma:
 *   a = (p q)/(p + q); x = a * fma(Z,Z, fma(Y,Y, X*X)); F_0..F_L(x) as point_f64;
 *   R^{(k)}_{000} = ((-2a)^k, by repeated products) * F_k;
 *   R_{t,u,v} = fma(X, R_{t-1,u,v}, (t-1) * R_{t-2,u,v})  (t > 0; first term
 *   alone at t = 1), else the u then v recurrence; pref = ((2 pi^{5/2}) /
 *   ((p q) sqrt(p+q))) K_i K_j.  Output [Nb][Nk][NH].  Returns the first
 *   offending quartet index (x invalid or p, q <= 0), or -1. */
static int herm_count(int L) { return (L + 1) * (L + 2) * (L + 3) / 6; }
static int herm_index(int t, int u, int v) {
  const int s = t + u + v;
  int before = 0;
  for (int tp = s; tp > t; --tp) before += s - tp + 1;
  return herm_count(s - 1) + before + (s - t - u);
}

int64_t boys_oracle_hermite(const void* tab, int L, const double* bra, int64_t Nb,
                            const double* ket, int64_t Nk, double* out) {
  const oracle_table* ot = tab;
  if (L < 0 || L > 8) return -2;
  const int NH = herm_count(L);
  int64_t first_bad = INT64_MAX;
  const double two_pi52 = 0x1.17e50a9dc6553p+5;   /* RN(2 pi^{5/2}) */
#pragma omp parallel for schedule(static) reduction(min : first_bad)
  for (int64_t q = 0; q < Nb * Nk; ++q) {
    const double* b = bra + 5 * (q / Nk);
    const double* k = ket + 5 * (q % Nk);
    const double p = b[0], qq = k[0];
    const double X = b[1] - k[1], Y = b[2] - k[2], Z = b[3] - k[3];
    const double pq = p + qq;
    const double a = (p * qq) / pq;
    const double r2 = fma(Z, Z, fma(Y, Y, X * X));
    const double x = a * r2;
    double F[MAXN + 1], R[165], R0[MAXN + 1] = {0};
    int ok = point_f64(&ot->t64, L, x, F, NULL);
    if (!(p > 0.0 && qq > 0.0)) {
      ok = 0;
      for (int m = 0; m <= L; ++m) F[m] = NAN;
    }
    const double m2a = -2.0 * a;
    double pw = 1.0;
    for (int m = 0; m <= L; ++m) {
      R0[m] = pw * F[m];
      pw = pw * m2a;
    }
    R[0] = R0[L];
    for (int n = L - 1; n >= 0; --n) {
      for (int s = L - n; s >= 1; --s)
        for (int t = s; t >= 0; --t)
          for (int u = s - t; u >= 0; --u) {
            const int v = s - t - u;
            double val;
            if (t > 0)
              val = t >= 2 ? fma(X, R[herm_index(t - 1, u, v)], (double)(t - 1) * R[herm_index(t - 2, u, v)])
                           : X * R[herm_index(t - 1, u, v)];
            else if (u > 0)
              val = u >= 2 ? fma(Y, R[herm_index(0, u - 1, v)], (double)(u - 1) * R[herm_index(0, u - 2, v)])
                           : Y * R[herm_index(0, u - 1, v)];
            else
              val = v >= 2 ? fma(Z, R[herm_index(0, 0, v - 1)], (double)(v - 1) * R[herm_index(0, 0, v - 2)])
                           : Z * R[herm_index(0, 0, v - 1)];
            R[herm_index(t, u, v)] = val;
          }
      R[0] = R0[n];
    }
    const double den = (p * qq) * sqrt(pq);
    const double pref = ((two_pi52 / den) * b[4]) * k[4];
    for (int m = 0; m < NH; ++m) out[q * NH + m] = pref * R[m];
    if (!ok && q < first_bad) first_bad = q;
  }
  return first_bad == INT64_MAX ? -1 : first_bad;
}

/* Q~_n(x) alone (eval_qtilde), for SPEC.md:295-297 checks. */
void boys_oracle_qtilde(const void* t, int n, const void* x, int64_t N, void* out) {
  const oracle_table* ot = t;
  for (int64_t i = 0; i < N; ++i) {
    if (ot->is_f32) ((float*)out)[i] = qtilde_f32(&ot->t32.row[n], ((const float*)x)[i]);
    else ((double*)out)[i] = qtilde_f64(&ot->t64.row[n], ((const double*)x)[i]);
  }
}

/* e^{-x} of the shared exp algorithm (for its own accuracy test). */
void boys_oracle_expneg(int is_f32, const void* x, int64_t N, void* out) {
  init_consts_f64();
  init_consts_f32();
  for (int64_t i = 0; i < N; ++i) {
    if (is_f32) ((float*)out)[i] = exp_neg_clamped_f32(((const float*)x)[i]);
    else ((double*)out)[i] = exp_neg_clamped_f64(((const double*)x)[i]);
  }
}

int boys_oracle_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
