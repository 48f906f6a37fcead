/*
 * libboys -- B200-native batched Boys-function evaluator (arXiv 2504.07637).
 *
 * C ABI (extern "C", plain pointers and sizes, no torch types).  Every entry
 * point replaces a piece of the reference's SPEC'd kernel interface; the
 * reference ships it only as a specification, so each comment cites the SPEC
 * line that defines the behaviour and the refmath line that fixes the output
 * semantics (index m <-> F_m, recursion F_m = (2x F_{m+1} + e^-x)/(2m+1)).
 *
 *   reference interface                                  replaced by
 *   ---------------------------------------------------  -------------------------
 *   kernel.eval_batch(EvalRequest{n, xs, layout}, T)      boys_eval_dense
 *       SPEC.md:316-324; semantics refmath.py:330-341
 *   kernel.eval_fn(n, x, T) -> (fn, expx)                 boys_eval_dense(n_max=n,
 *       SPEC.md:298-306                                     expx_dev != NULL)
 *   kernel.eval_with_split(n, n_bar, x, T)                boys_eval_split
 *       SPEC.md:325-333
 *   ragged batches (per-element order)   boys_eval_ragged
 *   domain error "listing offending indices"              boys_domain_result
 *       SPEC.md:302, 320, 347; refmath.py:111-115
 *   order check (refmath.py:104-108, MAX_ORDER :41)       BOYS_E_ORDER / boys_max_order
 *   eval_batch with host arrays (the CPU caller's view)   boys_eval_dense_host
 *   ragged work lists with host arrays                   boys_eval_ragged_host
 *   downstream integral code (SURVEY     boys_hermite_coulomb
 *       8(f)#4: fused consumer of F_m)
 *
 * Conventions
 *   - Device pointers are caller-owned, 16-byte aligned for x/out, and the work
 *     is stream-ordered on `stream` (a cudaStream_t passed as void*; NULL =
 *     legacy default stream).  No allocation and no host sync on the device
 *     entry points; tables are compiled into the module (__constant__).
 *     Kernels launch with programmatic stream serialization: a launch may
 *     begin (and boys_eval_dense at n_max = 0 may read x and evaluate) while
 *     the stream's previous kernel is still draining, but it writes nothing
 *     before that kernel has completed, and it re-reads x afterwards and
 *     re-evaluates if a value changed -- results are those of a fully
 *     serialized launch.  x must be a mapped device buffer when the call is
 *     made (it always is for memory the caller owns at that point).
 *   - Layouts: BOYS_SOA = order-major [n_max+1][N]; BOYS_AOS = point-major
 *     [N][n_max+1] ("order-major, point-major").
 *   - Domain: x must be finite and >= 0 (-0.0 is accepted as 0).  Offending
 *     elements produce NaN outputs; if `dom_dev` is non-NULL the smallest
 *     offending index is atomically min-reduced into it.  The caller
 *     initialises *dom_dev to -1 (all bits set) = "no error".
 *   - Results are bit-identical to the CPU restatement in oracle/ (same
 *     operation sequence, explicit FMA, IEEE div/sqrt, shared exp algorithm).
 */
#ifndef BOYS_H_
#define BOYS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BOYS_OK = 0,
  BOYS_E_DOMAIN = 1,  /* some x < 0, NaN or inf (only from *_host / domain_result) */
  BOYS_E_ORDER = 2,   /* n_max < 0 or above boys_max_order(dtype) */
  BOYS_E_LAYOUT = 3,
  BOYS_E_DTYPE = 4,
  BOYS_E_ALIGN = 5,   /* x/out not 16-byte aligned, or bad sizes */
  BOYS_E_CUDA = 6,    /* CUDA runtime error (see boys_last_cuda_error) */
  BOYS_E_ARG = 7      /* NULL pointer / negative N / bad split */
} boys_status;

typedef enum { BOYS_F64 = 0, BOYS_F32 = 1 } boys_dtype;
typedef enum { BOYS_SOA = 0, BOYS_AOS = 1 } boys_layout;

/* Highest tabulated order for the dtype (36 for f64, 16 for f32). */
int boys_max_order(boys_dtype dtype);

/* Library / table version string ("libboys <ver> tables <sha-prefix>"). */
const char* boys_version(void);

/* F_0..F_{n_max}(x_i) for i < N into out_dev (layout as above).
 * expx_dev (nullable): e^{-x_i} as used by the recursion (0 for x > 708 in f64, x > 86 in f32). */
boys_status boys_eval_dense(boys_dtype dtype, int n_max, const void* x_dev, int64_t N,
                            void* out_dev, boys_layout layout, void* expx_dev,
                            int64_t* dom_dev, void* stream);

/* Ragged batch: element i has its own order nmax_dev[i] (0..boys_max_order)
 * and writes F_0..F_{n_i} to out_dev[offsets_dev[i] + m]; offsets_dev has N+1
 * entries (exclusive prefix sum of n_i + 1).  Values are bit-identical to
 * boys_eval_dense at order n_i for the same x. */
boys_status boys_eval_ragged(boys_dtype dtype, const void* x_dev, const uint8_t* nmax_dev,
                             const int64_t* offsets_dev, int64_t N, void* out_dev,
                             int64_t* dom_dev, void* stream);

/* offsets_dev[0] = 0, offsets_dev[i+1] = offsets_dev[i] + nmax_dev[i] + 1. */
boys_status boys_ragged_offsets(const uint8_t* nmax_dev, int64_t N, int64_t* offsets_dev,
                                void* stream);

/* eval_with_split: F_n seeds the recursion n -> n_bar+1 and
 * an independent F_{n_bar} seeds n_bar -> 0.  0 <= n_bar < n. */
boys_status boys_eval_split(boys_dtype dtype, int n, int n_bar, const void* x_dev, int64_t N,
                            void* out_dev, boys_layout layout, int64_t* dom_dev, void* stream);

/* Synchronises `stream`, copies *dom_dev to *first_bad (-1 = all valid). */
boys_status boys_domain_result(const int64_t* dom_dev, int64_t* first_bad, void* stream);

/* Host-buffer entry (end-to-end path): x_host[N] -> out_host in `layout`,
 * pipelined host->device copy / kernel / device->host copy over chunks on the
 * current device.  Blocks until done.  Host buffers should be pinned for full
 * link speed.  Returns BOYS_E_DOMAIN (and *first_bad) if some x is invalid. */
boys_status boys_eval_dense_host(boys_dtype dtype, int n_max, const void* x_host, int64_t N,
                                 void* out_host, boys_layout layout, int64_t* first_bad);

/* Host-buffer ragged entry (end-to-end path for ragged batches): x_host[N] and
 * nmax_host[N] -> out_host, element i's F_0..F_{n_i} at its exclusive prefix
 * offset sum_{j<i}(n_j + 1), pipelined over chunks (host->device copies, the
 * device offsets scan, the ragged kernel, device->host copy).  out_capacity:
 * values out_host holds (BOYS_E_ARG if below sum(n_i + 1)).  Blocks until
 * done.  BOYS_E_DOMAIN (and *first_bad) for an invalid x or an order above
 * boys_max_order.  Replaces the reference's host-side batch call for ragged
 * work lists (SPEC.md:316-324 with per-element orders). */
boys_status boys_eval_ragged_host(boys_dtype dtype, const void* x_host, const uint8_t* nmax_host,
                                  int64_t N, void* out_host, int64_t out_capacity,
                                  int64_t* first_bad);

/* ---- coefficient tables (eval_batch(req, KernelTable),
 * eval_with_split(n, n_bar, x, table), table loading from the coeffs file) ----
 * The compiled-in tables serve boys_eval_dense / _split / _ragged.  A caller
 * holding a different KernelTable (a refit, another dataset file) uploads it
 * once and evaluates through the *_table entries; values are bit-identical to
 * the CPU restatement loaded with that dataset.  Row layout: BoysRow<T> of
 * csrc/boys_eval.cuh (q0 q1 q2 c z x_up, uq[8][2], ul[2], vq[8][2], vl[2] in
 * the dtype, then int32 cnt[4]), boys_table_row_bytes(dtype) bytes per order. */
typedef struct boys_table boys_table;

/* SHA-256 (hex) of the compiled table's packed rows (coeffs.table_checksum). */
const char* boys_table_checksum(boys_dtype dtype);
size_t boys_table_row_bytes(boys_dtype dtype);
/* Upload rows for orders 0..n_rows-1 to the current device (synchronous). */
boys_status boys_table_create(boys_dtype dtype, const void* rows_host, int n_rows,
                              size_t row_bytes, boys_table** out);
boys_status boys_table_destroy(boys_table* table);
int boys_table_max_order(const boys_table* table);
boys_status boys_eval_dense_table(const boys_table* table, int n_max, const void* x_dev,
                                  int64_t N, void* out_dev, boys_layout layout, void* expx_dev,
                                  int64_t* dom_dev, void* stream);
boys_status boys_eval_split_table(const boys_table* table, int n, int n_bar, const void* x_dev,
                                  int64_t N, void* out_dev, boys_layout layout,
                                  int64_t* dom_dev, void* stream);

/* Per-shard error statistic (the multi-GPU path's only reduction):
 * *err_dev = max(*err_dev, max_j |(vals[pos_j] - hi_j) - lo_j| / max(|hi_j|, tiny))
 * over j < K, gold_dev = K (hi, lo) double-double reference pairs, tiny = the
 * dtype's smallest normal (absolute error below it); NaN contributes +inf.  Stream-ordered,
 * one launch; the caller initialises *err_dev (0.0) and gathers it across ranks. */
boys_status boys_shard_error(boys_dtype dtype, const void* vals_dev, const int64_t* pos_dev,
                             const double* gold_dev, int64_t K, double* err_dev, void* stream);

/* Fused consumer (the downstream integral code SPEC.md:16, 353
 * names as the caller): McMurchie-Davidson Hermite Coulomb integrals for every
 * (bra pair i, ket pair j), F_0..F_L evaluated in registers and consumed there:
 *   a = p q/(p+q), x = a |P-Q|^2, R^{(n)}_{000} = (-2a)^n F_n(x), Helgaker's
 *   recurrences to R^{(0)}_{tuv}, t+u+v <= L;
 *   out[(i Nk + j) NH + k] = 2 pi^{5/2} / (p q sqrt(p+q)) K_i K_j R_{tuv},
 * NH = (L+1)(L+2)(L+3)/6 in the canonical order (s = t+u+v ascending, then t
 * descending, then u descending).  Pair records are 5 doubles: p, Px, Py, Pz, K.
 * 0 <= L <= 4 (BOYS_E_ORDER otherwise); fp64; stream-ordered.  dom_dev: first
 * quartet with an invalid x or p, q <= 0 (their outputs are NaN). */
boys_status boys_hermite_coulomb(int L, const double* bra_dev, int64_t Nb, const double* ket_dev,
                                 int64_t Nk, double* out_dev, int64_t* dom_dev, void* stream);

/* Number of kernel launches issued by this library in this process. */
int64_t boys_launch_count(void);

const char* boys_status_str(boys_status s);
const char* boys_last_cuda_error(void);

#ifdef __cplusplus
}
#endif
#endif /* BOYS_H_ */
