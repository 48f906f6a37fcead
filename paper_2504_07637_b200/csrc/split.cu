// eval_with_split: two seeds, two recursions.  Part of libboys.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <type_traits>

#include "boys_device.cuh"
#include "boys_launch.h"

namespace boys {

// SoA split: 3 resident blocks (80 registers); unbounded (134 registers, 1
// block) was 2x slower
constexpr int kSplitSoaMinB = 3;

// ---------------------------------------------------------------------------
// split kernel (eval_with_split): F_m for m <= nbar equals a
// dense order-nbar evaluation, F_m for m > nbar a dense order-n evaluation.
// One e^{-x} per point serves both seeds; the order-n recursion stops at
// nbar + 1 (its lower values are never used).  NBAR >= 0: compile-time lower
// order (the common pairs); NBAR < 0: run-time nbar (uniform loops).
// ---------------------------------------------------------------------------
template <typename T, int n, int NBAR, typename Put>
__device__ __forceinline__ void split_point(T x_in, bool ok, int nbar_rt, Put&& put) {
  using A = Ar<T>;
  const int nbar = NBAR >= 0 ? NBAR : nbar_rt;      // warp-uniform
  const T x = ok ? x_in : A::nan();                  // NaN through every step
  const T t = exp_neg_select(x);
  const T tx = A::add(x, x);
  {
    // order n: seed, recursion n-1 .. nbar+1
    const BoysRow<T>& R = Tab<T>::row(n);
    T cur = seed<T, n>(x, t, __any_sync(kFull, ok && x < R.z));
    put(n, cur);
#pragma unroll
    for (int m = n - 1; m >= 0; --m) {
      if (m <= nbar) break;
      cur = A::mul(A::fma(tx, cur, t), rinv<T>(m));
      put(m, cur);
    }
  }
  if constexpr (NBAR >= 0) {
    // order nbar (compile time): seed, recursion nbar-1 .. 0
    const BoysRow<T>& R = Tab<T>::row(NBAR);
    T cur = seed<T, NBAR>(x, t, __any_sync(kFull, ok && x < R.z));
    put(NBAR, cur);
#pragma unroll
    for (int m = NBAR - 1; m >= 0; --m) {
      cur = A::mul(A::fma(tx, cur, t), rinv<T>(m));
      put(m, cur);
    }
  } else {
    // order nbar (run time, uniform): the operation sequence of seed<T, nbar>
    constexpr int MQ = MaxShape<T>::Q(), ML = MaxShape<T>::L();
    const BoysRow<T>& R = Tab<T>::row(nbar);
    const int bits = 32 - __clz(nbar | 1);
    T y = x;
    if (__any_sync(kFull, ok && x < R.z)) {
      const T u = factored_uniform<T, MQ, ML>(x, R.uq, R.ul, R.cnt[0], R.cnt[1]);
      const T v = factored_uniform<T, MQ, ML>(x, R.vq, R.vl, R.cnt[2], R.cnt[3]);
      T h = A::mul(R.q2, A::div(u, v));
      h = A::fma(h, x, R.q1);
      const T Q = A::fma(h, x, R.q0);
      const T sq = A::sqrt(Q);
      const T s = nbar == 0 ? sq : A::mul(powi_rt_bounded(Q, nbar, bits), sq);
      const T yq = A::fma(s, t, x);
      y = x < R.z ? yq : x;
    }
    const T r = A::rcp(y);
    const T sr = A::sqrt(r);
    T cur = A::mul(A::mul(R.c, powi_rt_bounded(r, nbar, bits)), sr);   // nbar = 0: c * 1.0 == c
    put(nbar, cur);
#pragma unroll
    for (int m = n - 2; m >= 0; --m) {
      if (m < nbar) {
        cur = A::mul(A::fma(tx, cur, t), rinv<T>(m));
        put(m, cur);
      }
    }
  }
  // upward ladder past x_up (order-n values above nbar, order-nbar ones below)
  const bool up_hi = ok && x > Tab<T>::row(n).x_up;
  const bool up_lo = ok && x > Tab<T>::row(nbar).x_up;
  if (__any_sync(kFull, up_hi || up_lo)) {
    const T rx = A::rcp(x);
    T f = up_first(x);
    if (up_lo) put(0, f);
#pragma unroll
    for (int m = 0; m < n; ++m) {
      f = up_next(f, m, rx);
      if (m + 1 <= nbar ? up_lo : up_hi) put(m + 1, f);
    }
  }
}

template <typename T, int n, int NBAR, bool AOS, int NBUF>
__global__ void __launch_bounds__(kThreads, AOS ? 4 : kSplitSoaMinB)
split_kernel(const T* __restrict__ X, int64_t N, int nbar, T* __restrict__ out,
             int64_t* __restrict__ dom, bool bulk_ok) {
  constexpr int W = n + 1, WS = RowStride<W>::value;
  constexpr int TILE_ELEMS = kThreads * WS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* sbase = reinterpret_cast<T*>(smem_raw);
  const int tid = threadIdx.x;
  const int64_t ntiles = (N + kThreads - 1) / kThreads;
  pdl_wait_and_release();
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int64_t i0 = tile * kThreads;
    const int64_t i = i0 + tid;
    const bool in = i < N;
    const T x = in ? ldg_nc(X + i) : T(0);
    bool ok = valid_x(x);
    if (in && !ok) flag_domain(dom, i);
    ok = ok || !in;
    if constexpr (AOS) {
      // as the dense AoS path: [256][n+1] tile staged in shared memory (odd
      // row stride: conflict-free), one bulk copy per tile, NBUF-deep
      T* buf = sbase + (it % NBUF) * TILE_ELEMS;
      if (tid == 0) bulk_wait_read<NBUF - 1>();
      __syncthreads();
      T* row = buf + tid * WS;
      split_point<T, n, NBAR>(x, ok, nbar, [&](int m, T v) { row[m] = v; });
      const int64_t cnt = (N - i0) < kThreads ? (N - i0) : kThreads;
      if (!RowStride<W>::padded && bulk_ok && cnt == kThreads) {
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) bulk_store(out + i0 * W, buf, TILE_ELEMS * sizeof(T));
      } else {
        __syncthreads();
        copy_out_rows<T, W, WS>(out + i0 * W, buf, cnt, tid, kThreads);
      }
    } else {
      T* o = out + i;
      split_point<T, n, NBAR>(x, ok, nbar, [&](int m, T v) {
        if (in) __stcs(o + (int64_t)m * N, v);
      });
    }
  }
  if (AOS && tid == 0) bulk_wait_all();
}

template <typename T, int n, bool AOS>
static boys_status launch_split_t(const T* x, int64_t N, int nbar, T* out, int64_t* dom,
                                  cudaStream_t s) {
  constexpr bool fits2 = 2 * kThreads * (n + 1) * sizeof(T) <= 80 * 1024 && !RowStride<n + 1>::padded;
  // double-buffered staging below n = 12; from there one buffer and four
  // resident blocks (two seeds per point: more warps pay more than the second
  // buffer; same-box 2^24 points: (16, 8) 0.419 vs 0.429 ms, (12, 11) 0.357 vs
  // 0.361 ms, but (8, 4) 0.320 vs 0.318 ms)
  constexpr int NBUF = (AOS && fits2 && n < 12) ? 2 : 1;
  // compile-time lower order for the common pairs: n_bar = n - 1 (one more
  // order: "a few more bits") and n_bar = n / 2
  // (orders above 16 only run-time nbar: compile time and library size)
  constexpr bool SPEC = n <= 16;
  constexpr int NB1 = SPEC ? n - 1 : -1, NB2 = SPEC ? n / 2 : -1;
  const int var = (SPEC && nbar == NB1) ? 0 : (SPEC && nbar == NB2) ? 1 : 2;
  auto k = var == 0   ? split_kernel<T, n, NB1, AOS, NBUF>
           : var == 1 ? split_kernel<T, n, NB2, AOS, NBUF>
                      : split_kernel<T, n, -1, AOS, NBUF>;
  const size_t smem = AOS ? (size_t)NBUF * kThreads * RowStride<n + 1>::value * sizeof(T) : 0;
  static std::atomic<uint64_t> attr_mask[3];         // per kernel variant, per device
  if (AOS) {
    boys_status st = opt_in_smem(k, (int)smem, attr_mask[var]);
    if (st != BOYS_OK) return st;
  }
  const int64_t ntiles = (N + kThreads - 1) / kThreads;
  const bool bulk_ok = (reinterpret_cast<uintptr_t>(out) % 16) == 0;
  k<<<blocks_for(k, smem, ntiles), kThreads, smem, s>>>(x, N, nbar, out, dom, bulk_ok);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_status(cudaGetLastError());
}

template <typename T, int n = 1>
static boys_status dispatch_split(int nn, int nbar, const void* x, int64_t N, void* out,
                                  boys_layout lay, int64_t* dom, cudaStream_t s) {
  if constexpr (n > Tab<T>::MAX_ORDER) {
    return BOYS_E_ORDER;
  } else {
    if (nn == n) {
      if (lay == BOYS_AOS) return launch_split_t<T, n, true>((const T*)x, N, nbar, (T*)out, dom, s);
      return launch_split_t<T, n, false>((const T*)x, N, nbar, (T*)out, dom, s);
    }
    return dispatch_split<T, n + 1>(nn, nbar, x, N, out, lay, dom, s);
  }
}

boys_status eval_split_base(boys_dtype dtype, int n, int n_bar, const void* x, int64_t N,
                            void* out, boys_layout lay, int64_t* dom, cudaStream_t s) {
  if (dtype == BOYS_F64) return dispatch_split<double>(n, n_bar, x, N, out, lay, dom, s);
  return dispatch_split<float>(n, n_bar, x, N, out, lay, dom, s);
}

}  // namespace boys
