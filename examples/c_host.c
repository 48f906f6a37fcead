/* A plain C caller of libboys through include/boys.h only (no CUDA headers,
 * no torch): the host-buffer entries, as a compiled host of the reference's
 * batch interface would bind them.
 *
 *   gcc -O2 -std=c11 -I include examples/c_host.c \
 *       -L paper_2504_07637_b200 -lboys -Wl,-rpath,$PWD/paper_2504_07637_b200 -o c_host
 *   ./c_host x.bin n.bin out_dense.bin out_ragged.bin N
 *
 * x.bin: N float64; n.bin: N uint8 orders.  Writes F_0..F_16 point-major for
 * every x (boys_eval_dense_host) and the ragged F_0..F_{n_i}
 * (boys_eval_ragged_host).  Exit status = the first non-OK boys_status. */
#include <stdio.h>
#include <stdlib.h>

#include "boys.h"

static void* slurp(const char* path, size_t bytes) {
  FILE* f = fopen(path, "rb");
  if (!f) return NULL;
  void* p = malloc(bytes ? bytes : 1);
  size_t got = fread(p, 1, bytes, f);
  fclose(f);
  if (got != bytes) { free(p); return NULL; }
  return p;
}

static int spill(const char* path, const void* p, size_t bytes) {
  FILE* f = fopen(path, "wb");
  if (!f) return -1;
  size_t put = fwrite(p, 1, bytes, f);
  fclose(f);
  return put == bytes ? 0 : -1;
}

int main(int argc, char** argv) {
  if (argc != 6) {
    fprintf(stderr, "usage: %s x.bin n.bin out_dense.bin out_ragged.bin N\n", argv[0]);
    return 64;
  }
  const int64_t N = atoll(argv[5]);
  double* x = slurp(argv[1], (size_t)N * sizeof(double));
  uint8_t* n = slurp(argv[2], (size_t)N);
  if (!x || !n) { fprintf(stderr, "cannot read inputs\n"); return 65; }
  printf("%s, max order %d (f64)\n", boys_version(), boys_max_order(BOYS_F64));

  double* dense = malloc((size_t)N * 17 * sizeof(double));
  int64_t bad = -1;
  boys_status st = boys_eval_dense_host(BOYS_F64, 16, x, N, dense, BOYS_AOS, &bad);
  if (st != BOYS_OK) { fprintf(stderr, "dense: %s (index %lld)\n", boys_status_str(st), (long long)bad); return st; }

  int64_t total = 0;
  for (int64_t i = 0; i < N; ++i) total += n[i] + 1;
  double* ragged = malloc((size_t)total * sizeof(double));
  st = boys_eval_ragged_host(BOYS_F64, x, n, N, ragged, total, &bad);
  if (st != BOYS_OK) { fprintf(stderr, "ragged: %s (index %lld)\n", boys_status_str(st), (long long)bad); return st; }

  /* the reference's errors: a negative x is a domain error naming its index */
  double neg[3] = {1.0, -2.0, 3.0};
  double tmp[3 * 17];
  st = boys_eval_dense_host(BOYS_F64, 16, neg, 3, tmp, BOYS_AOS, &bad);
  if (st != BOYS_E_DOMAIN || bad != 1) { fprintf(stderr, "domain check failed\n"); return 70; }
  st = boys_eval_dense_host(BOYS_F64, boys_max_order(BOYS_F64) + 1, x, 1, tmp, BOYS_AOS, &bad);
  if (st != BOYS_E_ORDER) { fprintf(stderr, "order check failed\n"); return 71; }

  if (spill(argv[3], dense, (size_t)N * 17 * sizeof(double)) ||
      spill(argv[4], ragged, (size_t)total * sizeof(double))) return 72;
  printf("ok: %lld dense rows, %lld ragged values\n", (long long)N, (long long)total);
  free(x); free(n); free(dense); free(ragged);
  return 0;
}
