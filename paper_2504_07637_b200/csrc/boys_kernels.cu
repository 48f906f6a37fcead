// sm_100a kernels and the C ABI of libboys (include/boys.h).
//
// dense  : persistent grid, one point per thread, 256-point tiles.
//          SoA  -> coalesced streaming stores, one row per order.
//          AoS  -> [256][n+1] tile staged in shared memory (odd row stride =>
//                  conflict-free 64-bit banks), then ONE bulk async copy
//                  (cp.async.bulk.global.shared::cta, TMA engine) per tile,
//                  double-buffered so the next tile computes while the
//                  previous one drains to HBM.
// ragged : per-element order; tables staged in shared memory, run-time-order
//          evaluator with exact select predication (bit-identical to dense),
//          output staged per block and written with coalesced stores.
// split  : eval_with_split (two seeds, two recursions).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/boys.h"
#include "boys_eval.cuh"

#ifndef BOYS_VERSION
#define BOYS_VERSION "0.1.0"
#endif

namespace boys {

constexpr int kThreads = 256;   // points per tile == threads per block

static std::atomic<int64_t> g_launches{0};
static thread_local char g_cuda_err[256] = "";

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
__device__ __forceinline__ void bulk_wait_read_le1() {
  asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

template <typename T> __device__ __forceinline__ T ldg_nc(const T* p) { return __ldg(p); }

// F_0..F_n for one point into Fv[]; returns false if x is outside the domain.
// `ok` lanes only influence warp-uniform shortcuts, never values.
template <typename T, int n>
__device__ __forceinline__ void eval_point(T x_in, bool ok, T (&Fv)[n + 1], T& t_out) {
  using A = Ar<T>;
  const BoysRow<T>& R = Tab<T>::row(n);
  T x = ok ? x_in : T(0);
  T t = exp_neg_clamped(x);
  bool below = ok && x < R.z;
  bool any_below = __any_sync(0xffffffffu, below);
  Fv[n] = seed<T, n>(x, t, any_below);
  T tx = A::add(x, x);
#pragma unroll
  for (int m = n - 1; m >= 0; --m) Fv[m] = A::mul(A::fma(tx, Fv[m + 1], t), rinv<T>(m));
  bool up = ok && x > R.x_up;
  if (__any_sync(0xffffffffu, up)) {
    T rx = A::rcp(x);
    T f = up_first(x);
    Fv[0] = up ? f : Fv[0];
#pragma unroll
    for (int m = 0; m < n; ++m) {
      f = up_next(f, m, rx);
      Fv[m + 1] = up ? f : Fv[m + 1];
    }
  }
  if (!ok) {
#pragma unroll
    for (int m = 0; m <= n; ++m) Fv[m] = A::nan();
    t = A::nan();
  }
  t_out = t;
}

// ---------------------------------------------------------------------------
// dense kernel
//
// Persistent grid over 256-point tiles, one point per thread, x of the next
// tile prefetched into registers while the current one computes.
// SoA: coalesced streaming stores per order row.
// AoS: each warp stages its 32 rows ([32][n+1], contiguous in global memory)
//      in its own shared-memory slot and issues its own bulk async copy
//      (TMA engine) -- no block-wide barrier; NBUF slots per warp rotate so
//      the copy of one tile overlaps the computation of the next.
// ---------------------------------------------------------------------------
enum : int { kPrefetch = 1, kWarpStore = 2 };

template <typename T, int n, bool AOS, int NBUF>
__global__ void __launch_bounds__(kThreads, (n <= 1 && !AOS) ? 8 : 4)
dense_kernel(const T* __restrict__ X, int64_t N, T* __restrict__ out, T* __restrict__ expx,
             int64_t* __restrict__ dom, int64_t index_base, bool bulk_ok, int flags) {
  constexpr int W = n + 1;
  constexpr int WARP_ELEMS = 32 * W;           // one warp's rows
  constexpr int TILE_ELEMS = kThreads * W;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool prefetch = flags & kPrefetch;
  const bool warp_store = flags & kWarpStore;
  T* sbase = reinterpret_cast<T*>(smem_raw);
  const int64_t ntiles = (N + kThreads - 1) / kThreads;
  int64_t tile = blockIdx.x;
  T x_next = T(0);
  if (prefetch && tile < ntiles && tile * kThreads + tid < N) x_next = ldg_nc(X + tile * kThreads + tid);
  int it = 0;
  for (; tile < ntiles; tile += gridDim.x, ++it) {
    const int64_t i0 = tile * kThreads;
    const int64_t i = i0 + tid;
    const bool in = i < N;
    T x;
    if (prefetch) {
      x = x_next;
      const int64_t inx = i + (int64_t)gridDim.x * kThreads;
      if (tile + gridDim.x < ntiles && inx < N) x_next = ldg_nc(X + inx);
    } else {
      x = in ? ldg_nc(X + i) : T(0);
    }
    bool ok = valid_x(x);
    if (in && !ok) flag_domain(dom, index_base + i);
    ok = ok || !in;   // tail lanes evaluate x = 0 quietly
    T Fv[W];
    T t;
    eval_point<T, n>(in ? x : T(0), ok, Fv, t);
    if (expx && in) __stcs(expx + i, t);
    if constexpr (!AOS) {
      if (in) {
#pragma unroll
        for (int m = 0; m < W; ++m) __stcs(out + (int64_t)m * N + i, Fv[m]);
      }
    } else if (warp_store) {
      // per-warp slot, per-warp bulk copy, no block barrier
      T* buf = sbase + warp * (NBUF * WARP_ELEMS) + (it % NBUF) * WARP_ELEMS;
      if (lane == 0) {
        if constexpr (NBUF == 1) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
        else asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
      }
      __syncwarp();
#pragma unroll
      for (int m = 0; m < W; ++m) buf[lane * W + m] = Fv[m];
      const int64_t w0 = i0 + warp * 32;
      const int64_t rows = N - w0 < 32 ? (N - w0 > 0 ? N - w0 : 0) : 32;
      if (bulk_ok && rows == 32) {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) bulk_store(out + w0 * W, buf, WARP_ELEMS * sizeof(T));
      } else {
        __syncwarp();
        T* dst = out + w0 * W;
        for (int k = lane; k < rows * W; k += 32) __stcs(dst + k, buf[k]);
      }
    } else {
      // block-wide tile, one bulk copy per tile
      T* buf = sbase + (it % NBUF) * TILE_ELEMS;
      if (tid == 0) {
        if constexpr (NBUF == 1) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
        else asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
      }
      __syncthreads();
#pragma unroll
      for (int m = 0; m < W; ++m) buf[tid * W + m] = Fv[m];
      const int64_t cnt = (N - i0) < kThreads ? (N - i0) : kThreads;
      if (bulk_ok && cnt == kThreads) {
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) bulk_store(out + i0 * W, buf, TILE_ELEMS * sizeof(T));
      } else {
        __syncthreads();
        T* dst = out + i0 * W;
        for (int k = tid; k < cnt * W; k += kThreads) __stcs(dst + k, buf[k]);
      }
    }
  }
  if constexpr (AOS) {
    if ((warp_store && lane == 0) || tid == 0) bulk_wait_all();
  }
}

// ---------------------------------------------------------------------------
// run-time-order evaluation (ragged / split)
// ---------------------------------------------------------------------------
template <typename T>
struct SmemTable {
  BoysRow<T> row[Tab<T>::MAX_ORDER + 1];
  int shape[Tab<T>::MAX_ORDER + 1][4];
};

template <typename T>
__device__ __forceinline__ void stage_table(SmemTable<T>& st) {
  const int words = sizeof(st.row) / sizeof(T);
  const T* src = reinterpret_cast<const T*>(&Tab<T>::row(0));
  T* dst = reinterpret_cast<T*>(&st.row[0]);
  for (int k = threadIdx.x; k < words; k += blockDim.x) dst[k] = src[k];
  for (int k = threadIdx.x; k < (Tab<T>::MAX_ORDER + 1) * 4; k += blockDim.x)
    (&st.shape[0][0])[k] = Tab<T>::shape(k / 4, k % 4);
}

// Seed F_n(x) for a run-time order n; identical operation sequence to seed<T,n>.
template <typename T, int MQ, int ML>
__device__ __forceinline__ T seed_rt(T x, T t, int n, const SmemTable<T>& st, bool any_below) {
  using A = Ar<T>;
  const BoysRow<T>& R = st.row[n];
  T y = x;
  if (any_below) {
    T u = factored_rt<T, MQ, ML>(x, R.uq, R.ul, st.shape[n][0], st.shape[n][1]);
    T v = factored_rt<T, MQ, ML>(x, R.vq, R.vl, st.shape[n][2], st.shape[n][3]);
    T w = A::div(u, v);
    T h = A::mul(R.q2, w);
    h = A::fma(h, x, R.q1);
    T Q = A::fma(h, x, R.q0);
    T sq = A::sqrt(Q);
    T s = n == 0 ? sq : A::mul(powi_rt(Q, n), sq);
    T yq = A::fma(s, t, x);
    y = x < R.z ? yq : x;
  }
  T r = A::rcp(y);
  T sr = A::sqrt(r);
  return n == 0 ? A::mul(R.c, sr) : A::mul(A::mul(R.c, powi_rt(r, n)), sr);
}

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

// Run-time order evaluation of F_0..F_n into Fv[0..n] (entries above n are
// unspecified).  Operation-for-operation the same as eval_point<T, n>.
template <typename T, int NB, int MQ, int ML>
__device__ __forceinline__ void eval_point_rt(T x_in, bool ok, int n, const SmemTable<T>& st,
                                              T (&Fv)[NB + 1], T& t_out) {
  using A = Ar<T>;
  T x = ok ? x_in : T(0);
  int ns = ok ? n : 0;
  T t = exp_neg_clamped(x);
  bool below = ok && x < st.row[ns].z;
  bool any_below = __any_sync(0xffffffffu, below);
  T cur = seed_rt<T, MQ, ML>(x, t, ns, st, any_below);
  Fv[NB] = cur;
  T tx = A::add(x, x);
#pragma unroll
  for (int m = NB - 1; m >= 0; --m) {
    T nx = A::mul(A::fma(tx, cur, t), rinv<T>(m));
    cur = m < ns ? nx : cur;
    Fv[m] = cur;
  }
  bool up = ok && x > st.row[ns].x_up;
  if (__any_sync(0xffffffffu, up)) {
    T rx = A::rcp(x);
    T f = up_first(x);
    Fv[0] = up ? f : Fv[0];
#pragma unroll
    for (int m = 0; m < NB; ++m) {
      f = up_next(f, m, rx);
      Fv[m + 1] = (up && m + 1 <= ns) ? f : Fv[m + 1];
    }
  }
  if (!ok) {
#pragma unroll
    for (int m = 0; m <= NB; ++m) Fv[m] = A::nan();
    t = A::nan();
  }
  t_out = t;
}

// ---------------------------------------------------------------------------
// ragged kernel: element i, order n_i, values at out[offsets[i] + m]
//
// Per 256-element tile:
//   stage    x, n, local output offset into shared memory; ballot-compact the
//            elements that need e^{-x} (x <= XEXP) and those below their
//            cut-off (x < z_{n_i}) into two lists; counting-sort the tile by
//            order n_i.
//   phase A  threads sweep the compacted lists: e^{-x}, then Q~ / s / y with
//            the run-time-order evaluator (per-lane tables from shared memory)
//            -- only ~28% / ~5% of ERI-like elements pay for these.
//   phase B  each thread takes one element of the order-sorted tile; a warp
//            loops over the (usually one or two) distinct orders it holds and
//            runs the compile-time-order tail (r = 1/y, F_n, recursion,
//            upward ladder) for that order, writing into the staged tile.
//   store    the tile's contiguous output range leaves with coalesced
//            streaming stores.
// Every value is bit-identical to boys_eval_dense at the element's order.
// Tiles holding an order above the table fall back to direct NaN writes.
// ---------------------------------------------------------------------------
// ragged v1: every lane runs the run-time-order evaluator (exact select
// predication to the compile-time bound NB); kept for A/B measurement.
template <typename T, int NB>
__global__ void __launch_bounds__(kThreads)
ragged_v1_kernel(const T* __restrict__ X, const uint8_t* __restrict__ NM,
                 const int64_t* __restrict__ OFF, int64_t N, T* __restrict__ out,
                 int64_t* __restrict__ dom) {
  using A = Ar<T>;
  constexpr int MQ = MaxShape<T>::Q(), ML = MaxShape<T>::L();
  __shared__ SmemTable<T> st;
  __shared__ T obuf[kThreads * (NB + 1)];
  stage_table(st);
  __syncthreads();
  const int tid = threadIdx.x;
  const int64_t ntiles = (N + kThreads - 1) / kThreads;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i0 = tile * kThreads;
    const int64_t i = i0 + tid;
    const bool in = i < N;
    const int64_t last = (i0 + kThreads < N) ? i0 + kThreads : N;
    const int64_t base = OFF[i0];
    const int64_t cnt = OFF[last] - base;
    T x = in ? ldg_nc(X + i) : T(0);
    const int n = in ? (int)NM[i] : 0;
    const int64_t off = in ? OFF[i] - base : 0;
    const bool xok = valid_x(x);
    if (in && !(xok && n <= NB)) flag_domain(dom, i);
    T Fv[NB + 1];
    T t;
    eval_point_rt<T, NB, MQ, ML>(x, xok || !in, n <= NB ? n : 0, st, Fv, t);
    const bool bad_tile = __syncthreads_or(in && n > NB);   // also: obuf free
    if (bad_tile) {
      if (in) {
        T* dst = out + base + off;
        for (int m = 0; m <= n; ++m) dst[m] = (n > NB || !xok) ? A::nan() : Fv[m <= NB ? m : NB];
      }
      continue;
    }
    if (in) {
#pragma unroll
      for (int m = 0; m <= NB; ++m)
        if (m <= n) obuf[off + m] = Fv[m];
    }
    __syncthreads();
    T* dst = out + base;
    for (int64_t k = tid; k < cnt; k += kThreads) __stcs(dst + k, obuf[k]);
  }
}

template <typename T, int NB>
struct RaggedSmem {
  SmemTable<T> st;
  T obuf[kThreads * (NB + 1)];
  T sx[kThreads], sy[kThreads], stt[kThreads];
  int soff[kThreads];
  int hist[NB + 2];
  short perm[kThreads];
  short listE[kThreads], listQ[kThreads];
  unsigned char sn[kThreads], sok[kThreads];
  int nE, nQ;
};

// F_n from y (= x past the cut-off) and the recursion/upward ladder, written
// to dst[0..n].  `mask` = lanes of this warp holding order n.
template <typename T, int n>
__device__ __forceinline__ void tail_store(T x, T y, T t, bool ok, unsigned mask, T* dst) {
  using A = Ar<T>;
  const BoysRow<T>& R = Tab<T>::row(n);
  T Fv[n + 1];
  T r = A::rcp(y);
  T sr = A::sqrt(r);
  Fv[n] = n == 0 ? A::mul(R.c, sr) : A::mul(A::mul(R.c, powi<T, (n == 0 ? 1 : n)>(r)), sr);
  T tx = A::add(x, x);
#pragma unroll
  for (int m = n - 1; m >= 0; --m) Fv[m] = A::mul(A::fma(tx, Fv[m + 1], t), rinv<T>(m));
  bool up = ok && x > R.x_up;
  if (__any_sync(mask, up)) {
    T rx = A::rcp(x);
    T f = up_first(x);
    Fv[0] = up ? f : Fv[0];
#pragma unroll
    for (int m = 0; m < n; ++m) {
      f = up_next(f, m, rx);
      Fv[m + 1] = up ? f : Fv[m + 1];
    }
  }
#pragma unroll
  for (int m = 0; m <= n; ++m) dst[m] = ok ? Fv[m] : A::nan();
}

template <typename T, int NB, int n = 0>
__device__ __forceinline__ void tail_dispatch(int nn, T x, T y, T t, bool ok, unsigned mask,
                                              T* dst) {
  if constexpr (n <= NB) {
    if (nn == n) tail_store<T, n>(x, y, t, ok, mask, dst);
    else tail_dispatch<T, NB, n + 1>(nn, x, y, t, ok, mask, dst);
  }
}

template <typename T, int NB>
__global__ void __launch_bounds__(kThreads)
ragged_kernel(const T* __restrict__ X, const uint8_t* __restrict__ NM,
              const int64_t* __restrict__ OFF, int64_t N, T* __restrict__ out,
              int64_t* __restrict__ dom) {
  using A = Ar<T>;
  constexpr int MQ = MaxShape<T>::Q(), ML = MaxShape<T>::L();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RaggedSmem<T, NB>& S = *reinterpret_cast<RaggedSmem<T, NB>*>(smem_raw);
  stage_table(S.st);
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t ntiles = (N + kThreads - 1) / kThreads;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i0 = tile * kThreads;
    const int64_t i = i0 + tid;
    const bool in = i < N;
    const int64_t last = (i0 + kThreads < N) ? i0 + kThreads : N;
    const int64_t base = __ldg(OFF + i0);
    const int64_t cnt = __ldg(OFF + last) - base;
    T x = in ? ldg_nc(X + i) : T(0);
    const int n = in ? (int)NM[i] : 0;
    const int64_t off = in ? __ldg(OFF + i) - base : 0;
    const bool xok = valid_x(x);
    if (in && !(xok && n <= NB)) flag_domain(dom, i);
    if (tid < NB + 2) S.hist[tid] = 0;
    if (tid == 0) { S.nE = 0; S.nQ = 0; }
    __syncthreads();   // previous tile fully stored; table staged (first pass)
    if (__syncthreads_or(in && n > NB)) {
      // invalid order somewhere in the tile: direct writes, NaN for the bad ones
      if (in) {
        T* dst = out + base + off;
        if (n > NB || !xok) {
          for (int m = 0; m <= n; ++m) dst[m] = A::nan();
        } else {
          T Fv[NB + 1], t;
          eval_point_rt<T, NB, MQ, ML>(x, true, n, S.st, Fv, t);
          for (int m = 0; m <= n; ++m) dst[m] = Fv[m];
        }
      } else {
        T Fv[NB + 1], t;
        eval_point_rt<T, NB, MQ, ML>(T(0), true, 0, S.st, Fv, t);   // keep warps converged
      }
      continue;
    }
    const bool ok = in && xok;
    const T xs = ok ? x : T(0);
    const bool needE = ok && xs <= A::XEXP;
    const bool needQ = ok && xs < S.st.row[n].z;
    // stage + compaction (warp-aggregated atomics)
    S.sx[tid] = xs;
    S.sy[tid] = xs;
    S.stt[tid] = T(0);
    S.sn[tid] = (unsigned char)n;
    S.sok[tid] = ok;
    S.soff[tid] = (int)off;
    {
      unsigned bE = __ballot_sync(0xffffffffu, needE), bQ = __ballot_sync(0xffffffffu, needQ);
      int baseE = 0, baseQ = 0;
      if (lane == 0) {
        baseE = atomicAdd(&S.nE, __popc(bE));
        baseQ = atomicAdd(&S.nQ, __popc(bQ));
      }
      baseE = __shfl_sync(0xffffffffu, baseE, 0);
      baseQ = __shfl_sync(0xffffffffu, baseQ, 0);
      unsigned lt = (1u << lane) - 1u;
      if (needE) S.listE[baseE + __popc(bE & lt)] = (short)tid;
      if (needQ) S.listQ[baseQ + __popc(bQ & lt)] = (short)tid;
    }
    int rank_in_bin = in ? atomicAdd(&S.hist[n], 1) : 0;
    __syncthreads();
    // phase A1: e^{-x} on the compacted list
    for (int k = tid; k < S.nE; k += kThreads) {
      int e = S.listE[k];
      S.stt[e] = exp_neg_clamped(S.sx[e]);
    }
    if (tid == 0) {   // exclusive scan of the order histogram
      int acc = 0;
      for (int b = 0; b <= NB; ++b) {
        int h = S.hist[b];
        S.hist[b] = acc;
        acc += h;
      }
    }
    __syncthreads();
    // phase A2: y = x + Q~^{n+1/2} e^{-x} for elements below their cut-off
    for (int k = tid; k < S.nQ; k += kThreads) {
      int e = S.listQ[k];
      int ne = S.sn[e];
      const BoysRow<T>& R = S.st.row[ne];
      T xe = S.sx[e];
      T u = factored_rt<T, MQ, ML>(xe, R.uq, R.ul, S.st.shape[ne][0], S.st.shape[ne][1]);
      T v = factored_rt<T, MQ, ML>(xe, R.vq, R.vl, S.st.shape[ne][2], S.st.shape[ne][3]);
      T w = A::div(u, v);
      T h = A::mul(R.q2, w);
      h = A::fma(h, xe, R.q1);
      T Q = A::fma(h, xe, R.q0);
      T sq = A::sqrt(Q);
      T s = ne == 0 ? sq : A::mul(powi_rt(Q, ne), sq);
      S.sy[e] = A::fma(s, S.stt[e], xe);
    }
    if (in) S.perm[S.hist[n] + rank_in_bin] = (short)tid;
    __syncthreads();
    // phase B: order-sorted tails
    const int cntE = (int)(last - i0);
    const bool has = tid < cntE;
    const int e = has ? S.perm[tid] : 0;
    const int ne = has ? S.sn[e] : 0;
    unsigned todo = __ballot_sync(0xffffffffu, has);
    while (todo) {
      const int nl = __shfl_sync(0xffffffffu, ne, __ffs(todo) - 1);
      const bool mine = has && ne == nl;
      const unsigned mask = __ballot_sync(0xffffffffu, mine);
      if (mine)
        tail_dispatch<T, NB>(nl, S.sx[e], S.sy[e], S.stt[e], S.sok[e] != 0, mask,
                             S.obuf + S.soff[e]);
      todo &= ~mask;
    }
    __syncthreads();
    T* dst = out + base;
    for (int k = tid; k < (int)cnt; k += kThreads) __stcs(dst + k, S.obuf[k]);
  }
}

// ---------------------------------------------------------------------------
// split kernel (eval_with_split): F_m for m <= nbar equals a
// dense order-nbar evaluation, F_m for m > nbar a dense order-n evaluation.
// ---------------------------------------------------------------------------
template <typename T, int n, bool AOS>
__global__ void __launch_bounds__(kThreads)
split_kernel(const T* __restrict__ X, int64_t N, int nbar, T* __restrict__ out,
             int64_t* __restrict__ dom) {
  constexpr int W = n + 1;
  constexpr int MQ = MaxShape<T>::Q(), ML = MaxShape<T>::L();
  __shared__ SmemTable<T> st;
  stage_table(st);
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < N; i0 += stride) {
    const int64_t i = i0 + threadIdx.x;
    const bool in = i < N;
    T x = in ? ldg_nc(X + i) : T(0);
    bool ok = valid_x(x);
    if (in && !ok) flag_domain(dom, i);
    ok = ok || !in;
    T Fv[W], Fl[W];
    T t, tl;
    eval_point<T, n>(in ? x : T(0), ok, Fv, t);
    eval_point_rt<T, n, MQ, ML>(in ? x : T(0), ok, nbar, st, Fl, tl);
    if (in) {
#pragma unroll
      for (int m = 0; m < W; ++m) {
        T val = m <= nbar ? Fl[m] : Fv[m];
        if (AOS) __stcs(out + i * W + m, val);
        else __stcs(out + (int64_t)m * N + i, val);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// ragged offsets: exclusive prefix sum of (n_i + 1), single-pass per block +
// a tiny second pass over block totals (decoupled; two launches)
// ---------------------------------------------------------------------------
__global__ void offsets_block_kernel(const uint8_t* __restrict__ NM, int64_t N,
                                     int64_t* __restrict__ OFF, int64_t* __restrict__ blk) {
  __shared__ int64_t s[kThreads];
  const int64_t per = 8;
  const int64_t b0 = (int64_t)blockIdx.x * kThreads * per;
  int64_t loc[8];
  int64_t acc = 0;
  for (int k = 0; k < per; ++k) {
    int64_t i = b0 + threadIdx.x * per + k;
    loc[k] = acc;
    acc += (i < N) ? (int64_t)NM[i] + 1 : 0;
  }
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int d = 1; d < kThreads; d <<= 1) {
    int64_t v = threadIdx.x >= d ? s[threadIdx.x - d] : 0;
    __syncthreads();
    s[threadIdx.x] += v;
    __syncthreads();
  }
  int64_t excl = s[threadIdx.x] - acc;
  for (int k = 0; k < per; ++k) {
    int64_t i = b0 + threadIdx.x * per + k;
    if (i < N) OFF[i] = excl + loc[k];
  }
  if (threadIdx.x == kThreads - 1) blk[blockIdx.x] = s[threadIdx.x];
}

__global__ void offsets_fix_kernel(int64_t N, int64_t nblk, int64_t* __restrict__ OFF,
                                   const int64_t* __restrict__ blk) {
  // every block redundantly scans the block totals it needs (nblk is small)
  __shared__ int64_t add;
  const int64_t per = 8;
  const int64_t b = blockIdx.x;
  if (threadIdx.x == 0) {
    int64_t a = 0;
    for (int64_t k = 0; k < b; ++k) a += blk[k];
    add = a;
  }
  __syncthreads();
  const int64_t b0 = b * kThreads * per;
  for (int k = 0; k < per; ++k) {
    int64_t i = b0 + threadIdx.x * per + k;
    if (i < N) OFF[i] += add;
  }
  if (b == nblk - 1 && threadIdx.x == 0) {
    int64_t a = 0;
    for (int64_t k = 0; k < nblk; ++k) a += blk[k];
    OFF[N] = a;
  }
}

// ---------------------------------------------------------------------------
// launch plumbing
// ---------------------------------------------------------------------------
static int sm_count() {
  static int sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return sms;
}

static boys_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return BOYS_OK;
  snprintf(g_cuda_err, sizeof g_cuda_err, "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
  return BOYS_E_CUDA;
}

// Persistent grid (SMs x resident blocks) for large batches; for small ones
// (<= 4 waves) one block per tile so the block scheduler balances the tail.
template <typename K>
static int blocks_for(K kernel, size_t smem, int64_t ntiles) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, smem);
  if (occ < 1) occ = 1;
  int64_t b = (int64_t)sm_count() * occ;
  if (ntiles <= 4 * b) b = ntiles;
  return (int)(b < 1 ? 1 : b);
}

// Tuning knobs (read once; defaults are the measured best on B200):
//   BOYS_AOS_NBUF    staging depth (1 or 2)
//   BOYS_DENSE_FLAGS bit0 prefetch next tile's x, bit1 per-warp bulk stores
//   BOYS_RAGGED_V    ragged kernel variant (1 = predicated, 2 = compacted/sorted)
static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}
static int aos_nbuf() {
  static int v = env_int("BOYS_AOS_NBUF", 2) == 1 ? 1 : 2;
  return v;
}
static int dense_flags() {
  static int v = env_int("BOYS_DENSE_FLAGS", 0);
  return v;
}
static int ragged_variant() {
  static int v = env_int("BOYS_RAGGED_V", 2);
  return v;
}

template <typename T, int n, bool AOS, int NBUF>
static boys_status launch_dense_k(const T* x, int64_t N, T* out, T* expx, int64_t* dom,
                                  int64_t base, cudaStream_t s) {
  auto k = dense_kernel<T, n, AOS, NBUF>;
  size_t smem = AOS ? (size_t)NBUF * kThreads * (n + 1) * sizeof(T) : 0;
  static bool attr = false;   // per instantiation
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e);
    attr = true;
  }
  int64_t ntiles = (N + kThreads - 1) / kThreads;
  bool bulk_ok = (reinterpret_cast<uintptr_t>(out) % 16) == 0;
  k<<<blocks_for(k, smem, ntiles), kThreads, smem, s>>>(x, N, out, expx, dom, base, bulk_ok,
                                                        dense_flags());
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_status(cudaGetLastError());
}

template <typename T, int n, bool AOS>
static boys_status launch_dense_t(const T* x, int64_t N, T* out, T* expx, int64_t* dom,
                                  int64_t base, cudaStream_t s) {
  if (AOS && aos_nbuf() == 1) return launch_dense_k<T, n, AOS, 1>(x, N, out, expx, dom, base, s);
  return launch_dense_k<T, n, AOS, 2>(x, N, out, expx, dom, base, s);
}

template <typename T, int n>
static boys_status dispatch_dense_layout(const void* x, int64_t N, void* out, boys_layout lay,
                                         void* expx, int64_t* dom, int64_t base, cudaStream_t s) {
  if (lay == BOYS_AOS)
    return launch_dense_t<T, n, true>((const T*)x, N, (T*)out, (T*)expx, dom, base, s);
  return launch_dense_t<T, n, false>((const T*)x, N, (T*)out, (T*)expx, dom, base, s);
}

template <typename T, int n = 0>
static boys_status dispatch_dense(int nmax, const void* x, int64_t N, void* out, boys_layout lay,
                                  void* expx, int64_t* dom, int64_t base, cudaStream_t s) {
  if constexpr (n > Tab<T>::MAX_ORDER) {
    return BOYS_E_ORDER;
  } else {
    if (nmax == n) return dispatch_dense_layout<T, n>(x, N, out, lay, expx, dom, base, s);
    return dispatch_dense<T, n + 1>(nmax, x, N, out, lay, expx, dom, base, s);
  }
}

static boys_status eval_dense_base(boys_dtype dtype, int n_max, const void* x, int64_t N,
                                   void* out, boys_layout lay, void* expx, int64_t* dom,
                                   int64_t base, cudaStream_t s) {
  if (dtype == BOYS_F64) return dispatch_dense<double>(n_max, x, N, out, lay, expx, dom, base, s);
  return dispatch_dense<float>(n_max, x, N, out, lay, expx, dom, base, s);
}

template <typename T, int n, bool AOS>
static boys_status launch_split_t(const T* x, int64_t N, int nbar, T* out, int64_t* dom,
                                  cudaStream_t s) {
  auto k = split_kernel<T, n, AOS>;
  int64_t ntiles = (N + kThreads - 1) / kThreads;
  k<<<blocks_for(k, 0, ntiles), kThreads, 0, s>>>(x, N, nbar, out, dom);
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

template <typename T>
static boys_status launch_ragged(const void* x, const uint8_t* nm, const int64_t* off, int64_t N,
                                 void* out, int64_t* dom, cudaStream_t s) {
  constexpr int NB = Tab<T>::MAX_ORDER;
  int64_t ntiles = (N + kThreads - 1) / kThreads;
  if (ragged_variant() == 1) {
    auto k = ragged_v1_kernel<T, NB>;
    k<<<blocks_for(k, 0, ntiles), kThreads, 0, s>>>((const T*)x, nm, off, N, (T*)out, dom);
  } else {
    auto k = ragged_kernel<T, NB>;
    const size_t smem = sizeof(RaggedSmem<T, NB>);
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return cuda_status(e);
      attr = true;
    }
    k<<<blocks_for(k, smem, ntiles), kThreads, smem, s>>>((const T*)x, nm, off, N, (T*)out, dom);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_status(cudaGetLastError());
}

static size_t dsize(boys_dtype d) { return d == BOYS_F64 ? 8 : 4; }

// ---------------------------------------------------------------------------
// host-buffer pipeline workspace (per device, grown on demand, reused)
// ---------------------------------------------------------------------------
struct HostPipe {
  int device = -1;
  size_t cap_x = 0, cap_out = 0;
  void* dx[2] = {nullptr, nullptr};
  void* dout[2] = {nullptr, nullptr};
  int64_t* ddom = nullptr;
  cudaStream_t st[2] = {nullptr, nullptr};
};
static std::mutex g_pipe_mu;
static std::vector<HostPipe> g_pipes;

static boys_status pipe_get(int dev, size_t bx, size_t bo, HostPipe** out) {
  for (auto& p : g_pipes)
    if (p.device == dev) { *out = &p; break; }
  if (!*out) {
    g_pipes.emplace_back();
    *out = &g_pipes.back();
    (*out)->device = dev;
    for (auto& s : (*out)->st) {
      cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      if (e != cudaSuccess) return cuda_status(e);
    }
    cudaError_t e = cudaMalloc(&(*out)->ddom, sizeof(int64_t));
    if (e != cudaSuccess) return cuda_status(e);
  }
  HostPipe* p = *out;
  if (bx > p->cap_x || bo > p->cap_out) {
    for (int k = 0; k < 2; ++k) {
      cudaFree(p->dx[k]);
      cudaFree(p->dout[k]);
      p->dx[k] = p->dout[k] = nullptr;
      cudaError_t e = cudaMalloc(&p->dx[k], bx);
      if (e == cudaSuccess) e = cudaMalloc(&p->dout[k], bo);
      if (e != cudaSuccess) return cuda_status(e);
    }
    p->cap_x = bx;
    p->cap_out = bo;
  }
  return BOYS_OK;
}

}  // namespace boys

using namespace boys;

extern "C" {

int boys_max_order(boys_dtype dtype) {
  if (dtype == BOYS_F64) return BOYS_F64_MAX_ORDER;
  if (dtype == BOYS_F32) return BOYS_F32_MAX_ORDER;
  return -1;
}

const char* boys_version(void) { return "libboys " BOYS_VERSION " sm_100a"; }

int64_t boys_launch_count(void) { return g_launches.load(); }

const char* boys_last_cuda_error(void) { return g_cuda_err; }

const char* boys_status_str(boys_status s) {
  switch (s) {
    case BOYS_OK: return "ok";
    case BOYS_E_DOMAIN: return "domain error: argument must be finite and >= 0";
    case BOYS_E_ORDER: return "order outside the tabulated range";
    case BOYS_E_LAYOUT: return "unknown layout";
    case BOYS_E_DTYPE: return "unknown dtype";
    case BOYS_E_ALIGN: return "pointer not 16-byte aligned";
    case BOYS_E_CUDA: return "CUDA error";
    case BOYS_E_ARG: return "invalid argument";
  }
  return "unknown status";
}

static boys_status check_common(boys_dtype dtype, int n_max, const void* x, int64_t N,
                                const void* out, boys_layout layout) {
  if (dtype != BOYS_F64 && dtype != BOYS_F32) return BOYS_E_DTYPE;
  if (layout != BOYS_SOA && layout != BOYS_AOS) return BOYS_E_LAYOUT;
  if (n_max < 0 || n_max > boys_max_order(dtype)) return BOYS_E_ORDER;
  if (N < 0) return BOYS_E_ARG;
  if (N > 0 && (!x || !out)) return BOYS_E_ARG;
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(out)) % dsize(dtype))
    return BOYS_E_ALIGN;
  return BOYS_OK;
}

boys_status boys_eval_dense(boys_dtype dtype, int n_max, const void* x_dev, int64_t N,
                            void* out_dev, boys_layout layout, void* expx_dev, int64_t* dom_dev,
                            void* stream) {
  boys_status st = check_common(dtype, n_max, x_dev, N, out_dev, layout);
  if (st != BOYS_OK || N == 0) return st;
  return eval_dense_base(dtype, n_max, x_dev, N, out_dev, layout, expx_dev, dom_dev, 0,
                         (cudaStream_t)stream);
}

boys_status boys_eval_split(boys_dtype dtype, int n, int n_bar, const void* x_dev, int64_t N,
                            void* out_dev, boys_layout layout, int64_t* dom_dev, void* stream) {
  boys_status st = check_common(dtype, n, x_dev, N, out_dev, layout);
  if (st != BOYS_OK) return st;
  if (n_bar < 0 || n_bar >= n) return BOYS_E_ARG;
  if (N == 0) return BOYS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == BOYS_F64) return dispatch_split<double>(n, n_bar, x_dev, N, out_dev, layout, dom_dev, s);
  return dispatch_split<float>(n, n_bar, x_dev, N, out_dev, layout, dom_dev, s);
}

boys_status boys_eval_ragged(boys_dtype dtype, const void* x_dev, const uint8_t* nmax_dev,
                             const int64_t* offsets_dev, int64_t N, void* out_dev,
                             int64_t* dom_dev, void* stream) {
  if (dtype != BOYS_F64 && dtype != BOYS_F32) return BOYS_E_DTYPE;
  if (N < 0) return BOYS_E_ARG;
  if (N == 0) return BOYS_OK;
  if (!x_dev || !nmax_dev || !offsets_dev || !out_dev) return BOYS_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == BOYS_F64) return launch_ragged<double>(x_dev, nmax_dev, offsets_dev, N, out_dev, dom_dev, s);
  return launch_ragged<float>(x_dev, nmax_dev, offsets_dev, N, out_dev, dom_dev, s);
}

boys_status boys_ragged_offsets(const uint8_t* nmax_dev, int64_t N, int64_t* offsets_dev,
                                void* stream) {
  if (N < 0 || !offsets_dev || (N > 0 && !nmax_dev)) return BOYS_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (N == 0) return cuda_status(cudaMemsetAsync(offsets_dev, 0, sizeof(int64_t), s));
  const int64_t per_blk = (int64_t)kThreads * 8;
  const int64_t nblk = (N + per_blk - 1) / per_blk;
  int64_t* blk = nullptr;
  cudaError_t e = cudaMallocAsync(&blk, nblk * sizeof(int64_t), s);
  if (e != cudaSuccess) return cuda_status(e);
  offsets_block_kernel<<<(unsigned)nblk, kThreads, 0, s>>>(nmax_dev, N, offsets_dev, blk);
  offsets_fix_kernel<<<(unsigned)nblk, kThreads, 0, s>>>(N, nblk, offsets_dev, blk);
  g_launches.fetch_add(2, std::memory_order_relaxed);
  e = cudaGetLastError();
  cudaFreeAsync(blk, s);
  return cuda_status(e);
}

boys_status boys_domain_result(const int64_t* dom_dev, int64_t* first_bad, void* stream) {
  if (!dom_dev || !first_bad) return BOYS_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(first_bad, dom_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return cuda_status(e);
}

boys_status boys_eval_dense_host(boys_dtype dtype, int n_max, const void* x_host, int64_t N,
                                 void* out_host, boys_layout layout, int64_t* first_bad) {
  boys_status st = check_common(dtype, n_max, x_host, N, out_host, layout);
  if (st != BOYS_OK) return st;
  if (first_bad) *first_bad = -1;
  if (N == 0) return BOYS_OK;
  std::lock_guard<std::mutex> lk(g_pipe_mu);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e);
  const size_t es = dsize(dtype);
  const int W = n_max + 1;
  const int64_t chunk = N < (int64_t(1) << 22) ? N : (int64_t(1) << 22);
  HostPipe* p = nullptr;
  st = pipe_get(dev, chunk * es, chunk * W * es, &p);
  if (st != BOYS_OK) return st;
  e = cudaMemsetAsync(p->ddom, 0xff, sizeof(int64_t), p->st[0]);
  if (e != cudaSuccess) return cuda_status(e);
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  cudaEventRecord(ev, p->st[0]);
  cudaStreamWaitEvent(p->st[1], ev, 0);
  const int64_t nchunks = (N + chunk - 1) / chunk;
  for (int64_t c = 0; c < nchunks && st == BOYS_OK; ++c) {
    const int k = (int)(c & 1);
    cudaStream_t s = p->st[k];
    const int64_t i0 = c * chunk;
    const int64_t cn = (N - i0) < chunk ? (N - i0) : chunk;
    e = cudaMemcpyAsync(p->dx[k], (const char*)x_host + i0 * es, cn * es, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) { st = cuda_status(e); break; }
    st = eval_dense_base(dtype, n_max, p->dx[k], cn, p->dout[k], layout, nullptr, p->ddom, i0, s);
    if (st != BOYS_OK) break;
    if (layout == BOYS_AOS) {
      e = cudaMemcpyAsync((char*)out_host + i0 * W * es, p->dout[k], cn * W * es,
                          cudaMemcpyDeviceToHost, s);
    } else {
      e = cudaMemcpy2DAsync((char*)out_host + i0 * es, N * es, p->dout[k], cn * es, cn * es, W,
                            cudaMemcpyDeviceToHost, s);
    }
    if (e != cudaSuccess) st = cuda_status(e);
  }
  for (auto s : p->st) {
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess && st == BOYS_OK) st = cuda_status(e);
  }
  cudaEventDestroy(ev);
  if (st != BOYS_OK) return st;
  int64_t bad = -1;
  e = cudaMemcpy(&bad, p->ddom, sizeof(int64_t), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_status(e);
  if (bad >= 0) {
    if (first_bad) *first_bad = bad;
    return BOYS_E_DOMAIN;
  }
  return BOYS_OK;
}

}  // extern "C"
