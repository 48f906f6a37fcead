// Device-side building blocks shared by the libboys kernels: bulk-copy and
// predication helpers, the compile-time-order evaluators (one point / two
// points per thread) and the run-time-order evaluators (ragged / split).
// All arithmetic follows boys_eval.cuh (bit-identical to the CPU oracle).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "../../include/boys.h"
#include "boys_eval.cuh"

namespace boys {

constexpr int kThreads = 256;   // points per tile == threads per block
constexpr int kRaggedFastOrders = 16;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void flag_domain(int64_t* dom, int64_t i) {
  if (dom) atomicMin(reinterpret_cast<unsigned long long*>(dom), (unsigned long long)i);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// bulk async copy smem -> global (TMA engine); bytes % 16 == 0, both 16B aligned
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst),
               "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
// the same with raw operands (global address, shared address, bytes)
__device__ __forceinline__ void bulk_store_u(uint64_t gdst, uint32_t ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst),
               "r"(ssrc), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
template <int PENDING>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(PENDING) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

template <typename T> __device__ __forceinline__ T ldg_nc(const T* p) { return __ldg(p); }
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
// L2 prefetch of the block's first x tile (`tile` elements from blockIdx.x *
// tile, one 32-byte sector per thread), issued BEFORE waiting on the stream's
// previous grid: a cache hint, safe whoever produces x (L2 is the point of
// coherence), so the first loads after the wait hit L2 with a warm TLB.  A
// stream of 2^20-point n = 0 launches: 8.29 -> 7.78 us per launch (before
// that config got its speculative kernel); cfg2 -0.7%.  Used by the two-point
// SoA kernel only: at 2^24 points it cost the four-point SoA kernel 1-4.5%
// (n = 3..5) and the persistent AoS kernels 0.2-1% (cfg3, cfg5).
template <typename T>
__device__ __forceinline__ void prefetch_first_tile(const T* X, int64_t N, int tile) {
  constexpr int PER = 32 / (int)sizeof(T);
  const int k = (int)threadIdx.x * PER;
  const int64_t i = (int64_t)blockIdx.x * tile + k;
  if (k < tile && i < N) prefetch_l2(X + i);
}

// Programmatic dependent launch (launches with the programmatic-serialization
// attribute): wait until the stream's previous grid has completed and its
// memory is visible (a no-op for a normally serialised launch), then allow
// the stream's next grid to be scheduled onto SM slots as ours free up --
// only its launch and prologue overlap our tail; it waits the same way.
__device__ __forceinline__ void pdl_wait_and_release() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

// Predicated move / shared store (inline PTX so the compiler keeps plain
// predication instead of a divergent branch per recursion step).
__device__ __forceinline__ void pmov(bool p, double& dst, double v) {
  asm("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q mov.b64 %0, %1; }" : "+d"(dst) : "d"(v), "r"((int)p));
}
__device__ __forceinline__ void pmov(bool p, float& dst, float v) {
  asm("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q mov.b32 %0, %1; }" : "+f"(dst) : "f"(v), "r"((int)p));
}
__device__ __forceinline__ void psts(bool p, double* a, double v) {
  asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q st.shared.f64 [%0], %1; }"
               :: "r"(smem_u32(a)), "d"(v), "r"((int)p) : "memory");
}
__device__ __forceinline__ void psts(bool p, int64_t* a, int64_t v) {
  asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q st.shared.b64 [%0], %1; }"
               :: "r"(smem_u32(a)), "l"(v), "r"((int)p) : "memory");
}
__device__ __forceinline__ void psts(bool p, float* a, float v) {
  asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q st.shared.f32 [%0], %1; }"
               :: "r"(smem_u32(a)), "f"(v), "r"((int)p) : "memory");
}



// Shared-memory row stride for a staged [points][W] AoS tile.  The 32 lanes
// write element m of 32 consecutive rows together; a row width that is a
// multiple of 16 elements puts them all in one or two banks (f64 n=15 ran at
// 49.6% of HBM, n=31 at 60.0%, f32 n=15 at 60.7%), so those rows are padded by
// one element and the tile leaves through coalesced thread stores instead of
// one bulk copy (86.8 / 87.5 / 73.2%).  Other widths keep the dense layout and
// the bulk copy: padding every even width measured worse (f64 n=9: 68.6 vs
// 91.7%), the thread copy-out costing more than the milder conflicts.
template <int W>
struct RowStride {
  static constexpr bool padded = W % 16 == 0;
  static constexpr int value = padded ? W + 1 : W;
};
template <typename T, int W, int WS>
__device__ __forceinline__ void copy_out_rows(T* __restrict__ dst, const T* buf, int64_t cnt,
                                              int tid, int nthreads) {
  for (int64_t k = tid; k < cnt * W; k += nthreads)
    __stcs(dst + k, buf[(k / W) * WS + (k % W)]);
}

// F_0..F_n for one point, handed to put(m, value) in the order n, n-1, .., 0
// (then, for lanes past x_up, 0..n again with the upward values).  Returns
// e^{-x}.  `ok` = x in the domain; other lanes produce NaN.  Lanes only
// influence warp-uniform shortcuts (skip Q~ / the upward ladder), never values.
template <typename T, int n, typename Put>
__device__ __forceinline__ T eval_point_stream(T x_in, bool ok, Put&& put) {
  using A = Ar<T>;
  const BoysRow<T>& R = Tab<T>::row(n);
  const T bad = A::nan();
  // invalid lanes carry x = NaN: every IEEE step then yields NaN on its own
  // (t = 0, y = r = F = NaN, the recursion stays NaN, the ladder test is
  // false) -- no per-value select; valid lanes are untouched
  T x = ok ? x_in : bad;
  T t = exp_neg_clamped(x);
  bool any_below = __any_sync(kFull, ok && x < R.z);
  T cur = seed<T, n>(x, t, any_below);
  put(n, cur);
  T tx = A::add(x, x);
#pragma unroll
  for (int m = n - 1; m >= 0; --m) {
    cur = A::mul(A::fma(tx, cur, t), rinv<T>(m));
    put(m, cur);
  }
  bool up = ok && x > R.x_up;
  // n = 0: the ladder's F_0 = c_0 sqrt(1/x) is the y = x seed itself
  if (n > 0 && __any_sync(kFull, up)) {
    T rx = A::rcp(x);
    T f = up_first(x);
    if (up) put(0, f);
#pragma unroll
    for (int m = 0; m < n; ++m) {
      f = up_next(f, m, rx);
      if (up) put(m + 1, f);
    }
  }
  return ok ? t : bad;
}

// Array form (split kernel).
template <typename T, int n>
__device__ __forceinline__ void eval_point(T x_in, bool ok, T (&Fv)[n + 1], T& t_out) {
  t_out = eval_point_stream<T, n>(x_in, ok, [&](int m, T v) { Fv[m] = v; });
}

// seed<double, n> for P points with the correctly rounded div / sqrt / rcp
// taken through their branch-free fast paths (boys_eval.cuh: ptxas's own fast
// path and range test, bit-identical to the intrinsics): one warp vote per
// operation decides whether any lane needs the intrinsic instead (then every
// point of the thread recomputes that operation with it), so the P chains
// interleave without a branch region per call.  The FP64-bound small orders'
// multi-point SoA kernels use it.
// COLD: the fallbacks as volatile asm (they cannot be speculated above their
// vote).  Same values either way; it is a code-generation choice measured per
// kernel (dense.cu), like the kernel rules there.
template <int n, int P, bool COLD = false>
__device__ __forceinline__ void seed_multi_fast(const double (&x)[P], const double (&t)[P],
                                                bool any_below, double (&F)[P]) {
  using A = Ar<double>;
  const BoysRow<double>& R = Tab<double>::row(n);
  constexpr int LU = Tab<double>::shape(n, 0), lu = Tab<double>::shape(n, 1);
  constexpr int LV = Tab<double>::shape(n, 2), lv = Tab<double>::shape(n, 3);
  double y[P];
#pragma unroll
  for (int j = 0; j < P; ++j) y[j] = x[j];
  if (any_below) {
    double w[P], Q[P], sq[P];
    bool slow = false;
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const double u = factored<double, LU, lu>(x[j], R.uq, R.ul);
      const double v = factored<double, LV, lv>(x[j], R.vq, R.vl);
      bool sj;
      w[j] = A::div_fast(u, v, sj);
      slow = slow || sj;
    }
    if (__any_sync(kFull, slow)) {               // (never for finite x >= 0 in practice)
#pragma unroll
      for (int j = 0; j < P; ++j)
        w[j] = A::div(factored<double, LU, lu>(x[j], R.uq, R.ul),
                      factored<double, LV, lv>(x[j], R.vq, R.vl));
    }
    slow = false;
#pragma unroll
    for (int j = 0; j < P; ++j) {
      double h = A::mul(R.q2, w[j]);
      h = A::fma(h, x[j], R.q1);
      Q[j] = A::fma(h, x[j], R.q0);
      bool sj;
      sq[j] = A::sqrt_fast(Q[j], sj);
      slow = slow || sj;
    }
    if (__any_sync(kFull, slow)) {
#pragma unroll
      for (int j = 0; j < P; ++j) sq[j] = COLD ? A::sqrt_cold(Q[j]) : A::sqrt(Q[j]);
    }
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const double s = n == 0 ? sq[j] : A::mul(powi<double, (n == 0 ? 1 : n)>(Q[j]), sq[j]);
      const double yq = A::fma(s, t[j], x[j]);
      y[j] = x[j] < R.z ? yq : x[j];
    }
  }
  double r[P], sr[P];
  bool slow = false;
#pragma unroll
  for (int j = 0; j < P; ++j) {
    bool sj;
    r[j] = A::rcp_fast(y[j], sj);
    slow = slow || sj;
  }
  if (__any_sync(kFull, slow)) {
#pragma unroll
    for (int j = 0; j < P; ++j) r[j] = COLD ? A::rcp_cold(y[j]) : A::rcp(y[j]);
  }
  slow = false;
#pragma unroll
  for (int j = 0; j < P; ++j) {
    bool sj;
    sr[j] = A::sqrt_fast(r[j], sj);
    slow = slow || sj;
  }
  if (__any_sync(kFull, slow)) {
#pragma unroll
    for (int j = 0; j < P; ++j) sr[j] = COLD ? A::sqrt_cold(r[j]) : A::sqrt(r[j]);
  }
#pragma unroll
  for (int j = 0; j < P; ++j)
    F[j] = n == 0 ? A::mul(R.c, sr[j])
                  : A::mul(A::mul(R.c, powi<double, (n == 0 ? 1 : n)>(r[j])), sr[j]);
}

// Two adjacent points per thread, evaluated in lockstep: per point the same
// operation sequence as eval_point_stream (so the same bits); put(m, a, b)
// receives F_m of both points at once so a SoA row takes one 16-byte store.
// The warp-uniform shortcuts see 64 points instead of 32 (values unchanged).
// P points per thread in lockstep (generalises eval_pair_stream; per point the
// same operation sequence as eval_point_stream).  put(m, v[P]) gets F_m of all
// P points; put1(j, m, v) the upward-ladder values of point j.
// ANYBAD: `any_bad` is a warp-uniform run-time flag, false only if every ok[]
// of the warp is true; the NaN selects for invalid points then sit behind one
// uniform branch instead of running for every point (the n = 0 speculative
// kernel).  Without ANYBAD the selects run per point, as before: the kernels
// that use that form measured faster with it (dense.cu).
template <typename T, int n, int P, bool FAST = false, bool ANYBAD = false, bool COLD = false,
          typename Put, typename Put1>
__device__ __forceinline__ void eval_multi_stream(const T (&xin)[P], const bool (&ok)[P],
                                                  T (&tout)[P], Put&& put, Put1&& put1,
                                                  bool any_bad = true) {
  using A = Ar<T>;
  const BoysRow<T>& R = Tab<T>::row(n);
  const T bad = A::nan();
  T x[P], t[P], cur[P], tx[P];
  bool below = false, up = false;
  if constexpr (ANYBAD) {
#pragma unroll
    for (int j = 0; j < P; ++j) x[j] = xin[j];
    if (any_bad) {
#pragma unroll
      for (int j = 0; j < P; ++j) x[j] = ok[j] ? xin[j] : bad;
    }
  }
#pragma unroll
  for (int j = 0; j < P; ++j) {
    if constexpr (!ANYBAD) x[j] = ok[j] ? xin[j] : bad;
    t[j] = FAST ? exp_neg_select(x[j]) : exp_neg_clamped(x[j]);
    below = below || (ok[j] && x[j] < R.z);
  }
  const bool any_below = __any_sync(kFull, below);
  if constexpr (FAST && sizeof(T) == 8) {
    seed_multi_fast<n, P, COLD>(x, t, any_below, cur);
  } else {
#pragma unroll
    for (int j = 0; j < P; ++j) cur[j] = seed<T, n>(x[j], t[j], any_below);
  }
  put(n, cur);
#pragma unroll
  for (int j = 0; j < P; ++j) tx[j] = A::add(x[j], x[j]);
#pragma unroll
  for (int m = n - 1; m >= 0; --m) {
#pragma unroll
    for (int j = 0; j < P; ++j) cur[j] = A::mul(A::fma(tx[j], cur[j], t[j]), rinv<T>(m));
    put(m, cur);
  }
#pragma unroll
  for (int j = 0; j < P; ++j) up = up || (ok[j] && x[j] > R.x_up);
  // n = 0: the ladder's F_0 = c_0 sqrt(1/x) is the y = x seed itself
  if (n > 0 && __any_sync(kFull, up)) {
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const bool upj = ok[j] && x[j] > R.x_up;
      T rx = A::rcp(x[j]);
      T f = up_first(x[j]);
      if (upj) put1(j, 0, f);
#pragma unroll
      for (int m = 0; m < n; ++m) {
        f = up_next(f, m, rx);
        if (upj) put1(j, m + 1, f);
      }
    }
  }
  if constexpr (ANYBAD) {
#pragma unroll
    for (int j = 0; j < P; ++j) tout[j] = t[j];
    if (any_bad) {
#pragma unroll
      for (int j = 0; j < P; ++j) tout[j] = ok[j] ? t[j] : bad;
    }
  } else {
#pragma unroll
    for (int j = 0; j < P; ++j) tout[j] = ok[j] ? t[j] : bad;
  }
}

template <typename T, int n, bool FAST = false, typename Put, typename Put1>
__device__ __forceinline__ void eval_pair_stream(T xa, T xb, bool oka, bool okb, T& ta_out,
                                                 T& tb_out, Put&& put, Put1&& put1) {
  using A = Ar<T>;
  const BoysRow<T>& R = Tab<T>::row(n);
  const T bad = A::nan();
  T x[2] = {oka ? xa : bad, okb ? xb : bad};
  const bool ok[2] = {oka, okb};
  T t[2], cur[2], tx[2];
  bool below = false, up = false;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    t[j] = FAST ? exp_neg_select(x[j]) : exp_neg_clamped(x[j]);
    below = below || (ok[j] && x[j] < R.z);
  }
  const bool any_below = __any_sync(kFull, below);
  if constexpr (FAST && sizeof(T) == 8) {
    seed_multi_fast<n, 2>(x, t, any_below, cur);
  } else {
#pragma unroll
    for (int j = 0; j < 2; ++j) cur[j] = seed<T, n>(x[j], t[j], any_below);
  }
  put(n, cur[0], cur[1]);
#pragma unroll
  for (int j = 0; j < 2; ++j) tx[j] = A::add(x[j], x[j]);
#pragma unroll
  for (int m = n - 1; m >= 0; --m) {
#pragma unroll
    for (int j = 0; j < 2; ++j) cur[j] = A::mul(A::fma(tx[j], cur[j], t[j]), rinv<T>(m));
    put(m, cur[0], cur[1]);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) up = up || (ok[j] && x[j] > R.x_up);
  // n = 0: the ladder's F_0 = c_0 sqrt(1/x) is the y = x seed itself
  if (n > 0 && __any_sync(kFull, up)) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const bool upj = ok[j] && x[j] > R.x_up;
      T rx = A::rcp(x[j]);
      T f = up_first(x[j]);
      if (upj) put1(j, 0, f);
#pragma unroll
      for (int m = 0; m < n; ++m) {
        f = up_next(f, m, rx);
        if (upj) put1(j, m + 1, f);
      }
    }
  }
  ta_out = oka ? t[0] : bad;
  tb_out = okb ? t[1] : bad;
}

// ---------------------------------------------------------------------------
// run-time-order evaluation (ragged / split)
// ---------------------------------------------------------------------------
// Row accessors for the run-time-order evaluator: rows staged in shared
// memory (ragged fast path: per-lane orders) or read from __constant__
// (split: warp-uniform order -> broadcast; rare high-order ragged chunks).
template <typename T, int R>
struct SmemTable {
  BoysRow<T> row[R];
};

template <typename T, int R>
__device__ __forceinline__ void stage_table(SmemTable<T, R>& st) {
  static_assert(sizeof(BoysRow<T>) % sizeof(int) == 0, "row layout");
  constexpr int words = R * sizeof(BoysRow<T>) / sizeof(int);
  const int* src = reinterpret_cast<const int*>(&Tab<T>::row(0));
  int* dst = reinterpret_cast<int*>(&st.row[0]);
  for (int k = threadIdx.x; k < words; k += blockDim.x) dst[k] = src[k];
}

template <typename T>
struct SmemRows {
  const BoysRow<T>* p;
  __device__ __forceinline__ const BoysRow<T>& operator()(int n) const { return p[n]; }
};
template <typename T>
struct PtrRows {   // rows in global memory (a table uploaded at run time)
  const BoysRow<T>* __restrict__ p;
  __device__ __forceinline__ const BoysRow<T>& operator()(int n) const { return p[n]; }
};
template <typename T>
struct ConstRows {
  __device__ __forceinline__ const BoysRow<T>& operator()(int n) const { return Tab<T>::row(n); }
};

template <typename T> struct MaxShape;   // compile-time bounds on factor counts
template <> struct MaxShape<double> {
  __host__ __device__ static constexpr int Q() {
    int m = 0;
    for (int n = 0; n <= BOYS_F64_MAX_ORDER; ++n)
      for (int k : {0, 2}) m = boys_shape_f64(n, k) > m ? boys_shape_f64(n, k) : m;
    return m;
  }
  __host__ __device__ static constexpr int L() {
    int m = 0;
    for (int n = 0; n <= BOYS_F64_MAX_ORDER; ++n)
      for (int k : {1, 3}) m = boys_shape_f64(n, k) > m ? boys_shape_f64(n, k) : m;
    return m;
  }
};
template <> struct MaxShape<float> {
  __host__ __device__ static constexpr int Q() {
    int m = 0;
    for (int n = 0; n <= BOYS_F32_MAX_ORDER; ++n)
      for (int k : {0, 2}) m = boys_shape_f32(n, k) > m ? boys_shape_f32(n, k) : m;
    return m;
  }
  __host__ __device__ static constexpr int L() {
    int m = 0;
    for (int n = 0; n <= BOYS_F32_MAX_ORDER; ++n)
      for (int k : {1, 3}) m = boys_shape_f32(n, k) > m ? boys_shape_f32(n, k) : m;
    return m;
  }
};

// y = x + Q~^{n+1/2} e^{-x} below the cut-off, run-time order; identical
// operation sequence to seed<T, n>'s Q~ branch.
template <typename T, typename Rows>
__device__ __forceinline__ T y_below_rt(T x, T t, int n, const Rows& rows) {
  using A = Ar<T>;
  constexpr int MQ = MaxShape<T>::Q(), ML = MaxShape<T>::L();
  const BoysRow<T>& R = rows(n);
  T u = factored_rt<T, MQ, ML>(x, R.uq, R.ul, R.cnt[0], R.cnt[1]);
  T v = factored_rt<T, MQ, ML>(x, R.vq, R.vl, R.cnt[2], R.cnt[3]);
  T w = A::div(u, v);
  T h = A::mul(R.q2, w);
  h = A::fma(h, x, R.q1);
  T Q = A::fma(h, x, R.q0);
  T sq = A::sqrt(Q);
  T s = n == 0 ? sq : A::mul(powi_rt(Q, n), sq);
  return A::fma(s, t, x);
}

// b^n for n < 2^bits (bits: warp-uniform bound); same products as powi<T,n>:
// starting from 1.0 and multiplying by (bit ? b^(2^j) : 1.0) is exact for the
// unset bits (x * 1.0 == x) and 1.0 * b^(2^j0) == b^(2^j0) for the first set
// bit, so the rounded product sequence is identical -- with one select per
// step instead of a select over a conditional product.
template <typename T>
__device__ __forceinline__ T powi_rt_bounded(T b, int n, int bits) {
  using A = Ar<T>;
  // j = 0: 1.0 * b == b exactly, so a select (n < 2^bits with bits >= 1)
  T r = (n & 1) ? b : T(1), p = b;
#pragma unroll
  for (int j = 1; j < 6; ++j) {
    if (j >= bits) break;
    p = A::mul(p, p);
    r = A::mul(r, ((n >> j) & 1) ? p : T(1));
  }
  return r;
}

// Tail for a run-time order n (per lane): F_n from y, then the recursion and
// the upward ladder, handed to put(m, v, on): `on` says whether m <= n, i.e.
// whether the value is one of this lane's outputs (callers store
// unconditionally to a scratch slot otherwise, so the loop stays branch-free).
// `wmax` = warp-uniform max order bounds the loops.
template <typename T, int NB, typename Rows, typename Put>
__device__ __forceinline__ void tail_rt(T x, T y, T t, int n, bool ok, int wmax,
                                        const Rows& rows, Put&& put) {
  using A = Ar<T>;
  const T bad = A::nan();
  const int bits = 32 - __clz(wmax | 1);
  T r = A::rcp(y);
  T sr = A::sqrt(r);
  const T c = rows(n).c;
  T cur = A::mul(A::mul(c, powi_rt_bounded(r, n, bits)), sr);   // n = 0: exact, see above
  put(n, ok ? cur : bad, true);
  T tx = A::add(x, x);
#pragma unroll
  for (int m = NB - 1; m >= 0; --m) {
    if (m < wmax) {                                // warp-uniform
      T nx = A::mul(A::fma(tx, cur, t), rinv<T>(m));
      const bool on = m < n;
      cur = on ? nx : cur;
      put(m, ok ? cur : bad, on);
    }
  }
  bool up = ok && x > rows(n).x_up;
  if (__any_sync(kFull, up)) {
    T rx = A::rcp(x);
    T f = up_first(x);
    if (up) put(0, f, true);
#pragma unroll
    for (int m = 0; m < NB; ++m) {
      if (m >= wmax) break;
      f = up_next(f, m, rx);
      if (up && m + 1 <= n) put(m + 1, f, true);
    }
  }
}

// Root-factored product with a warp-uniform run-time factor count: the
// active steps of factored_rt (same products, same order), skipping the
// inactive ones with a uniform branch instead of selecting them away.
template <typename T, int MQ, int ML>
__device__ __forceinline__ T factored_uniform(T x, const T (*q)[2], const T* l, int nq, int nl) {
  using A = Ar<T>;
  T acc = T(1);
  bool first = true;
#pragma unroll
  for (int k = 0; k < MQ; ++k) {
    if (k >= nq) break;
    T d = A::sub(x, q[k][0]);
    T f = A::fma(d, d, q[k][1]);
    acc = first ? f : A::mul(acc, f);
    first = false;
  }
#pragma unroll
  for (int k = 0; k < ML; ++k) {
    if (k >= nl) break;
    T f = A::sub(x, l[k]);
    acc = first ? f : A::mul(acc, f);
    first = false;
  }
  return acc;
}

// eval_point_rt for an order that is the same on every lane of the warp
// (split kernel): uniform loop bounds instead of per-lane selects.  Invalid
// lanes evaluate x = 0 at that order and output NaN, as in eval_point_rt.
template <typename T, int NB, typename Rows, typename Put>
__device__ __forceinline__ T eval_point_uniform(T x_in, bool ok, int n, const Rows& rows,
                                                Put&& put) {
  using A = Ar<T>;
  constexpr int MQ = MaxShape<T>::Q(), ML = MaxShape<T>::L();
  T x = ok ? x_in : T(0);
  T t = exp_neg_clamped(x);
  const BoysRow<T>& R = rows(n);
  bool below = ok && x < R.z;
  T y = x;
  if (__any_sync(kFull, below)) {
    T u = factored_uniform<T, MQ, ML>(x, R.uq, R.ul, R.cnt[0], R.cnt[1]);
    T v = factored_uniform<T, MQ, ML>(x, R.vq, R.vl, R.cnt[2], R.cnt[3]);
    T w = A::div(u, v);
    T h = A::mul(R.q2, w);
    h = A::fma(h, x, R.q1);
    T Q = A::fma(h, x, R.q0);
    T sq = A::sqrt(Q);
    T s = n == 0 ? sq : A::mul(powi_rt_bounded(Q, n, 32 - __clz(n | 1)), sq);
    T yq = A::fma(s, t, x);
    y = below ? yq : x;
  }
  tail_rt<T, NB>(x, y, t, n, ok, n, rows, [&](int m, T v, bool on) {
    if (on) put(m, v);
  });
  return ok ? t : A::nan();
}

// Complete run-time-order evaluation (split kernel; ragged fallback tiles).
template <typename T, int NB, typename Rows, typename Put>
__device__ __forceinline__ void eval_point_rt(T x_in, bool ok, int n, const Rows& rows,
                                              Put&& put) {
  using A = Ar<T>;
  T x = ok ? x_in : T(0);
  int ns = ok ? n : 0;
  T t = exp_neg_clamped(x);
  bool below = ok && x < rows(ns).z;
  T y = x;
  if (__any_sync(kFull, below)) {
    T yq = y_below_rt(x, t, ns, rows);
    y = below ? yq : x;
  }
  int wmax = __reduce_max_sync(kFull, (unsigned)ns);
  tail_rt<T, NB>(x, y, t, ns, ok, wmax, rows, [&](int m, T v, bool on) {
    if (on) put(m, v);
  });
}

}  // namespace boys
