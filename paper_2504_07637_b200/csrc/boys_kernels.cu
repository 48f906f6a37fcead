// sm_100a kernels and the C ABI of libboys (include/boys.h).
//
// dense  : each F_m is streamed to its destination as the recursion produces
//          it (no per-thread value array); launches use programmatic
//          dependent launch (griddepcontrol) to overlap back-to-back kernels.
//          SoA  -> paired kernel: two adjacent points per thread, 16-byte x
//                  loads and 16-byte streaming stores per F_m row, one block
//                  per 512-point tile (one point per thread for odd N /
//                  unaligned buffers).
//          AoS  -> persistent grid of 256-point tiles; the [256][n+1] tile is
//                  staged in shared memory (odd row stride => conflict-free
//                  64-bit banks) and leaves as ONE bulk async copy
//                  (cp.async.bulk.global.shared::cta, TMA engine) that
//                  overlaps the next tile's computation.
// ragged : per-element order.  Warp-autonomous chunks of 32*EPL elements:
//          past-cut-off elements run the run-time-order tail into a staging
//          slot (jump-table entry into the unrolled recursion), below-cut-off
//          ones go to a warp queue evaluated 32 at a time; each chunk's output
//          range leaves as one bulk async copy.
// split  : eval_with_split (two seeds, two recursions), AoS staged as dense.
// host   : host-buffer pipelines (H2D / kernel / D2H over chunks, two streams)
//          for dense and ragged work.
// All values are bit-identical to the CPU oracle (oracle/boys_oracle.c).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <vector>

#include "../../include/boys.h"
#include "boys_eval.cuh"

#ifndef BOYS_VERSION
#define BOYS_VERSION "0.2.0"
#endif

namespace boys {

constexpr int kThreads = 256;   // points per tile == threads per block
constexpr int kRaggedFastOrders = 16;
#ifndef BOYS_SOA_MINB
#define BOYS_SOA_MINB 4   // SoA resident-block target (register budget 64/thread)
#endif
constexpr unsigned kFull = 0xffffffffu;
#ifndef BOYS_PAIR_MINB_SMALL
#define BOYS_PAIR_MINB_SMALL 5   // paired SoA kernel, n <= 1: resident-block target (47 registers; cfg1 9.27 us vs 9.50 / 9.71 / 9.65 / 9.75 for 6 / 4 / 3 / 8)
#endif
#ifndef BOYS_PAIR_FASTCR
#define BOYS_PAIR_FASTCR 0   // 1: paired SoA kernel shares fast-path checks for div/sqrt/rcp (A/B: slower, spills: cfg1 10.7 vs 9.5 us)
#endif
#ifndef BOYS_FAST_CR
#define BOYS_FAST_CR 0   // 1: ragged chunks use the branch-free CR rcp/sqrt fast paths (A/B: f64 1.88 vs 1.83 ms, slower)
#endif

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
__device__ __forceinline__ void psts(bool p, float* a, float v) {
  asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q st.shared.f32 [%0], %1; }"
               :: "r"(smem_u32(a)), "f"(v), "r"((int)p) : "memory");
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
  if (__any_sync(kFull, up)) {
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

// seed<double, n> for two points with the correctly rounded div / sqrt / rcp
// taken through their branch-free fast paths (boys_eval.cuh, bit-identical to
// the intrinsics): one warp vote per operation decides whether any lane needs
// the intrinsic instead, so the two chains share one check per operation.
template <int n>
__device__ __forceinline__ void seed_pair(const double (&x)[2], const double (&t)[2],
                                          bool any_below, double (&F)[2]) {
  using A = Ar<double>;
  const BoysRow<double>& R = Tab<double>::row(n);
  double y[2] = {x[0], x[1]};
  if (any_below) {
    constexpr int LU = Tab<double>::shape(n, 0), lu = Tab<double>::shape(n, 1);
    constexpr int LV = Tab<double>::shape(n, 2), lv = Tab<double>::shape(n, 3);
    double u[2], v[2], w[2], Q[2], sq[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      u[j] = factored<double, LU, lu>(x[j], R.uq, R.ul);
      v[j] = factored<double, LV, lv>(x[j], R.vq, R.vl);
    }
    bool s0, s1;
    w[0] = A::div_fast(u[0], v[0], s0);
    w[1] = A::div_fast(u[1], v[1], s1);
    if (__any_sync(kFull, s0 || s1)) { w[0] = A::div(u[0], v[0]); w[1] = A::div(u[1], v[1]); }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      double h = A::mul(R.q2, w[j]);
      h = A::fma(h, x[j], R.q1);
      Q[j] = A::fma(h, x[j], R.q0);
    }
    sq[0] = A::sqrt_fast(Q[0], s0);
    sq[1] = A::sqrt_fast(Q[1], s1);
    if (__any_sync(kFull, s0 || s1)) { sq[0] = A::sqrt(Q[0]); sq[1] = A::sqrt(Q[1]); }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const double s = n == 0 ? sq[j] : A::mul(powi<double, (n == 0 ? 1 : n)>(Q[j]), sq[j]);
      const double yq = A::fma(s, t[j], x[j]);
      y[j] = x[j] < R.z ? yq : x[j];
    }
  }
  double r[2], sr[2];
  bool s0, s1;
  r[0] = A::rcp_fast(y[0], s0);
  r[1] = A::rcp_fast(y[1], s1);
  if (__any_sync(kFull, s0 || s1)) { r[0] = A::rcp(y[0]); r[1] = A::rcp(y[1]); }
  sr[0] = A::sqrt_fast(r[0], s0);
  sr[1] = A::sqrt_fast(r[1], s1);
  if (__any_sync(kFull, s0 || s1)) { sr[0] = A::sqrt(r[0]); sr[1] = A::sqrt(r[1]); }
#pragma unroll
  for (int j = 0; j < 2; ++j)
    F[j] = n == 0 ? A::mul(R.c, sr[j])
                  : A::mul(A::mul(R.c, powi<double, (n == 0 ? 1 : n)>(r[j])), sr[j]);
}

// Two adjacent points per thread, evaluated in lockstep: per point the same
// operation sequence as eval_point_stream (so the same bits); put(m, a, b)
// receives F_m of both points at once so a SoA row takes one 16-byte store.
// The warp-uniform shortcuts see 64 points instead of 32 (values unchanged).
template <typename T, int n, typename Put, typename Put1>
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
    t[j] = exp_neg_clamped(x[j]);
    below = below || (ok[j] && x[j] < R.z);
  }
  const bool any_below = __any_sync(kFull, below);
#if BOYS_PAIR_FASTCR
  if constexpr (sizeof(T) == 8) seed_pair<n>(x, t, any_below, cur);
  else
#endif
  {
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
  if (__any_sync(kFull, up)) {
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

// SoA dense kernel, two adjacent points per thread (512-point tiles): x comes
// in as one 16-byte load and every F_m row leaves as 16-byte streaming stores
// (512 contiguous bytes per warp instruction, half the store instructions).
// Requires N even and 16-byte aligned x/out/expx (host checks).
template <typename T, int n, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
dense_soa_pair_kernel(const T* __restrict__ X, int64_t N, T* __restrict__ out,
                      T* __restrict__ expx, int64_t* __restrict__ dom, int64_t index_base) {
  using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
  const int tid = threadIdx.x;
  constexpr int TILE = 2 * kThreads;
  const int64_t ntiles = (N + TILE - 1) / TILE;
  pdl_wait_and_release();
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i = tile * TILE + 2 * tid;     // even; N even => i + 1 < N iff i < N
    const bool in = i < N;
    V2 xv;
    if (in) xv = __ldg(reinterpret_cast<const V2*>(X + i));
    else { xv.x = T(0); xv.y = T(0); }
    bool oka = valid_x(xv.x), okb = valid_x(xv.y);
    if (in && !oka) flag_domain(dom, index_base + i);
    if (in && !okb) flag_domain(dom, index_base + i + 1);
    oka = oka || !in;
    okb = okb || !in;
    T* o = out + i;
    T ta, tb;
    eval_pair_stream<T, n>(
        xv.x, xv.y, oka, okb, ta, tb,
        [&](int m, T a, T b) {
          V2 v;
          v.x = a;
          v.y = b;
          if (in) __stcs(reinterpret_cast<V2*>(o + (int64_t)m * N), v);
        },
        [&](int j, int m, T v) {
          if (in) __stcs(o + (int64_t)m * N + j, v);
        });
    if (expx && in) {
      V2 tv;
      tv.x = ta;
      tv.y = tb;
      __stcs(reinterpret_cast<V2*>(expx + i), tv);
    }
  }
}

// ---------------------------------------------------------------------------
// dense kernel
// ---------------------------------------------------------------------------
template <typename T, int n, bool AOS, int NBUF, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
dense_kernel(const T* __restrict__ X, int64_t N, T* __restrict__ out, T* __restrict__ expx,
             int64_t* __restrict__ dom, int64_t index_base, bool bulk_ok, bool soa_bulk) {
  constexpr int W = n + 1;
  constexpr int TILE_ELEMS = kThreads * W;
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
    // (loading the next tile's x one iteration ahead measured slower:
    // SoA 77% vs 84%, AoS 86% vs 94% of HBM, tools/ab/ab25.sh)
    const T x = in ? ldg_nc(X + i) : T(0);
    bool ok = valid_x(x);
    if (in && !ok) flag_domain(dom, index_base + i);
    ok = ok || !in;   // tail lanes evaluate x = 0 quietly
    if constexpr (!AOS) {
      if (soa_bulk) {
        // [n+1][256] tile in shared memory, one bulk copy per order row
        T* buf = sbase + (it % NBUF) * TILE_ELEMS;
        if (tid == 0) bulk_wait_read<NBUF - 1>();
        __syncthreads();
        T t = eval_point_stream<T, n>(x, ok, [&](int m, T v) { buf[m * kThreads + tid] = v; });
        if (expx && in) __stcs(expx + i, t);
        const int64_t cnt = (N - i0) < kThreads ? (N - i0) : kThreads;
        if (cnt == kThreads) {
          fence_proxy_async_smem();
          __syncthreads();
          if (tid < W) bulk_store(out + (int64_t)tid * N + i0, buf + tid * kThreads,
                                  kThreads * sizeof(T));
        } else {
          __syncthreads();
          for (int k = tid; k < W * kThreads; k += kThreads) {
            const int m = k / kThreads, j = k % kThreads;
            if (j < cnt) __stcs(out + (int64_t)m * N + i0 + j, buf[k]);
          }
        }
      } else {
        T* o = out + i;
        T t = eval_point_stream<T, n>(x, ok, [&](int m, T v) {
          if (in) __stcs(o + (int64_t)m * N, v);
        });
        if (expx && in) __stcs(expx + i, t);
      }
    } else {
      T* buf = sbase + (it % NBUF) * TILE_ELEMS;
      // the slot went to the bulk engine NBUF tiles ago: wait until it was read
      if (tid == 0) bulk_wait_read<NBUF - 1>();
      __syncthreads();
      T* row = buf + tid * W;
      T t = eval_point_stream<T, n>(x, ok, [&](int m, T v) { row[m] = v; });
      if (expx && in) __stcs(expx + i, t);
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
  if (AOS || soa_bulk) {
    if (tid < (AOS ? 1 : W)) bulk_wait_all();
  }
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
__device__ __forceinline__ void eval_point_uniform(T x_in, bool ok, int n, const Rows& rows,
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

// ---------------------------------------------------------------------------
// ragged kernel: element i, order n_i, values at out[offsets[i] + m]
//
// Warp-autonomous (no block barriers): each warp walks chunks of 32*EPL elements.
//   * every lane: e^{-x}; elements past their cut-off (x >= z_{n_i}, ~95% of
//     ERI-like batches) run the cheap run-time-order tail at once into the
//     warp's staging slot; the chunk's contiguous output range then leaves
//     with coalesced streaming stores (skipping deferred elements).
//   * elements below their cut-off are deferred to a warp-private queue and
//     evaluated 32 at a time with every lane busy (Q~ is the expensive part),
//     each lane writing its element's n+1 values directly.
// Values are bit-identical to boys_eval_dense at each element's order.
// ---------------------------------------------------------------------------
// EPL elements per lane (chunks of 32*EPL elements): the warp-uniform work of
// a chunk (ballots, jump-table dispatch, bulk store, constant loads) is shared
// by EPL elements per lane, whose independent chains also interleave (ILP).
// Staging holds CAP values; a chunk whose output range exceeds it takes the
// per-element direct-write path (never for ERI-like order mixes).
// CPE: staging values per element (NB + 1 = no overflow possible).
// MINB: __launch_bounds__ min blocks per SM (0 = unconstrained).
template <typename T, int NB, int EPL, int CPE>
struct RaggedWarp {
  static constexpr int CAP = 32 * EPL * (CPE < NB + 1 ? CPE : NB + 1);
  static constexpr int QCAP = 32 * EPL + 32;      // < 32 left after a drain + one chunk
  alignas(16) T stage[CAP + 16 / sizeof(T)];
  T qx[QCAP], qt[QCAP];
  int64_t qoff[QCAP];
  unsigned char qn[QCAP];
  T scratch[32];
};

template <typename T> struct alignas(4 * sizeof(T)) ZcRow { T z, c, x_up, pad; };  // per order

template <typename T, int NB, int EPL, int CPE, int WT = kThreads>
struct RaggedSmem {
  SmemTable<T, NB + 1> st;           // rows 0..NB (the fast path's orders)
  ZcRow<T> zc[NB + 1];               // per-order scalars, one 16/32-byte line each
  RaggedWarp<T, NB, EPL, CPE> w[WT / 32];
};

// Elements above x_up(n) (upward-ladder branch) join the queue in fp32, where
// x_up is low (2^7..2^60: ~2% of ERI-like elements; 1.00 vs 1.10 ms); in fp64
// x_up >= 2^60 and the chunk path keeps a (never taken) ladder, which
// measured 1.8% faster than queueing.
template <typename T> constexpr bool kDeferUp = sizeof(T) == 4;

// Evaluate up to 32 queued elements (one per lane), writing straight to
// global memory.
template <typename T, int NB, typename WarpT>
__device__ __forceinline__ void ragged_drain(WarpT& W, const SmemRows<T>& st,
                                             int& qn, int lane, T* __restrict__ out) {
  // queued elements' slots were written (with stale staging data) by earlier
  // bulk stores of their chunks: those must be complete before we overwrite
  if (lane == 0) bulk_wait_all();
  __syncwarp();
  const int take = qn < 32 ? qn : 32;
  const bool has = lane < take;
  const int slot = qn - take + lane;            // LIFO: drain the newest `take` entries
  const T x = has ? W.qx[slot] : T(0);
  const T t = has ? W.qt[slot] : T(0);
  const int n = has ? (int)W.qn[slot] : 0;
  const int64_t off = has ? W.qoff[slot] : 0;
  __syncwarp();
  // queued: below the cut-off (Q~ branch) or above x_up (asymptotic branch,
  // values from the upward ladder inside tail_rt)
  T y = x;
  if (kDeferUp<T>) {
    const bool below = has && x < st(n).z;
    if (__any_sync(kFull, below)) {
      const T yq = y_below_rt(x, t, n, st);
      y = below ? yq : x;
    }
  } else {
    y = has ? y_below_rt(x, t, n, st) : x;
  }
  const int wmax = __reduce_max_sync(kFull, (unsigned)n);
  T* dst = out + off;
  T* sink = W.scratch + lane;
  tail_rt<T, NB>(x, y, t, n, has, wmax, st,
                 [&](int m, T v, bool on) { *((has && on) ? dst + m : sink) = v; });
  qn -= take;
}

// Staging sentinel for deferred elements' slots: a NaN payload the arithmetic
// never produces (IEEE ops return the canonical quiet NaN).
template <typename T> struct Sentinel;
template <> struct Sentinel<double> {
  static __device__ __forceinline__ double value() { return __longlong_as_double(0x7ff4c0de5e47e1e1LL); }
  static __device__ __forceinline__ bool is(double v) { return __double_as_longlong(v) == 0x7ff4c0de5e47e1e1LL; }
};
template <> struct Sentinel<float> {
  static __device__ __forceinline__ float value() { return __int_as_float(0x7fa0c0de); }
  static __device__ __forceinline__ bool is(float v) { return __float_as_int(v) == 0x7fa0c0de; }
};

template <typename T, int NB, int EPL, int CPE, int MINB, int WT = kThreads>
__global__ void __launch_bounds__(WT, MINB)
ragged_kernel(const T* __restrict__ X, const uint8_t* __restrict__ NM,
              const int64_t* __restrict__ OFF, int64_t N, T* __restrict__ out,
              int64_t* __restrict__ dom) {
  using A = Ar<T>;
  using WarpT = RaggedWarp<T, NB, EPL, CPE>;
  constexpr int CH = 32 * EPL;                   // elements per chunk
  extern __shared__ __align__(128) unsigned char smem_raw[];
  using SmemT = RaggedSmem<T, NB, EPL, CPE, WT>;
  SmemT& S = *reinterpret_cast<SmemT*>(smem_raw);
  stage_table(S.st);
  for (int k = threadIdx.x; k <= NB; k += blockDim.x)
    S.zc[k] = ZcRow<T>{Tab<T>::row(k).z, Tab<T>::row(k).c, Tab<T>::row(k).x_up, T(0)};
  __syncthreads();
  const SmemRows<T> rows{S.st.row};
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpT& W = S.w[wid];
  const int64_t nchunks = (N + CH - 1) / CH;
  const int64_t wstride = (int64_t)gridDim.x * (WT / 32);
  int qn = 0;                                    // warp-uniform queue length
  int64_t c = (int64_t)blockIdx.x * (WT / 32) + wid;
  // software pipeline: inputs of chunk c are loaded one iteration ahead
  T px[EPL];
  int pn[EPL];
  int64_t poff[EPL], pbase = 0, plast_off = 0;
  int prem = 0;                                  // elements of the prefetched chunk
  auto load = [&](int64_t cc) {
    const int64_t j0 = cc * CH;
    if (j0 + CH <= N) {                          // full chunk (warp-uniform): no predicates
      prem = CH;
      const T* xp = X + j0 + lane;
      const uint8_t* np = NM + j0 + lane;
      const int64_t* op = OFF + j0 + lane;
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        px[e] = ldg_nc(xp + 32 * e);
        pn[e] = (int)np[32 * e];
        poff[e] = __ldg(op + 32 * e);
      }
    } else {
      // elements of chunk cc that exist (warp-uniform, 0 past the end)
      const int rem = cc < nchunks ? (int)(N - j0) : 0;
      prem = rem;
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        const int64_t j = j0 + 32 * e + lane;
        const bool jin = 32 * e + lane < rem;
        px[e] = jin ? ldg_nc(X + j) : T(0);
        pn[e] = jin ? (int)NM[j] : 0;
        poff[e] = jin ? __ldg(OFF + j) : 0;
      }
    }
    if (cc < nchunks) {
      pbase = __ldg(OFF + j0);
      plast_off = __ldg(OFF + ((j0 + CH < N) ? j0 + CH : N));
    }
  };
  load(c);
  for (; c < nchunks; c += wstride) {
    const int64_t i0 = c * CH;
    T x[EPL];
    int n[EPL];
    int64_t goff[EPL];
    bool in[EPL];
    const int rem = prem;
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      x[e] = px[e];
      n[e] = pn[e];
      goff[e] = poff[e];
      in[e] = 32 * e + lane < rem;
    }
    const int64_t base = pbase, cnt = plast_off - pbase;
    load(c + wstride);
    constexpr int MAXN = Tab<T>::MAX_ORDER;
    bool xok[EPL], slow = cnt > WarpT::CAP;
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      xok[e] = valid_x(x[e]);
      if (in[e] && !(xok[e] && n[e] <= MAXN)) flag_domain(dom, i0 + 32 * e + lane);
      slow = slow || (in[e] && n[e] > NB);
    }
    if (__any_sync(kFull, slow)) {
      // an order above the fast path's bound (or an output range above the
      // staging capacity): every lane evaluates its own elements from the
      // __constant__ rows and writes them directly (NaN above the table)
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        if (in[e] && n[e] > MAXN) {
          for (int m = 0; m <= n[e]; ++m) out[goff[e] + m] = A::nan();
        }
        const bool okl = in[e] && xok[e] && n[e] <= MAXN;
        T* dst = out + goff[e];
        const bool wd = in[e] && n[e] <= MAXN;
        eval_point_rt<T, MAXN>(x[e], okl, okl ? n[e] : 0, ConstRows<T>{}, [&](int m, T v) {
          if (wd) dst[m] = v;
        });
      }
      continue;
    }
    // staging position matches the global 16-byte phase of the chunk range
    constexpr int Q = 16 / sizeof(T);
    const int shift = (int)(base & (Q - 1));
    // the previous chunk's bulk store must have finished reading the slot
    if (lane == 0) bulk_wait_read<0>();
    __syncwarp();
    T xs[EPL], t[EPL], cur[EPL], tx[EPL];
    ZcRow<T> zc[EPL];
    T* dst[EPL];
    bool wr[EPL];
    int wmax_l = 0;
    // (evaluating e^{-x} only for the elements with x <= XEXP, compacted one
    // per lane, measured no faster: tools/ab/ab24.sh)
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      const bool ok = in[e] && xok[e];
      xs[e] = ok ? x[e] : A::nan();                // NaN propagates through the tail
      const T xe = ok ? x[e] : T(0);
      t[e] = exp_neg_clamped(xe);
      zc[e] = S.zc[n[e]];
      // deferred to the warp queue: below the cut-off (Q~ needed) and, in
      // fp32, above x_up (upward ladder)
      const bool defer = ok && (xe < zc[e].z || (kDeferUp<T> && xe > zc[e].x_up));
      const unsigned dmask = __ballot_sync(kFull, defer);
      dst[e] = W.stage + (int)(goff[e] - base) + shift;
      if (dmask) {                                 // enqueue (qn stays warp-uniform)
        if (defer) {
          const int slot = qn + __popc(dmask & ((1u << lane) - 1u));
          W.qx[slot] = xe;
          W.qt[slot] = t[e];
          W.qn[slot] = (unsigned char)n[e];
          W.qoff[slot] = goff[e];
        }
        qn += __popc(dmask);
      }
      wr[e] = in[e] && !defer;
      wmax_l = max(wmax_l, wr[e] ? n[e] : 0);
    }
    // immediate elements (past the cut-off): y = x.  Same operation sequence
    // as seed<T, n> + the recursion (+ the upward ladder in fp64).
    {
      const int wmax = __reduce_max_sync(kFull, (unsigned)wmax_l);
      const int bits = 32 - __clz(wmax | 1);
      T r[EPL], sr[EPL];
#if BOYS_FAST_CR
      // correctly rounded 1/x and sqrt through the branch-free fast paths for
      // all EPL elements at once (interleaved chains); the rare slow-path
      // lanes (x near 0 / the exponent limits, NaN) recompute with the intrinsics
      {
        bool slow = false;
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
          bool s1;
          r[e] = A::rcp_fast(xs[e], s1);
          slow = slow || s1;
        }
        if (__any_sync(kFull, slow)) {
#pragma unroll
          for (int e = 0; e < EPL; ++e) r[e] = A::rcp(xs[e]);
        }
        slow = false;
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
          bool s2;
          sr[e] = A::sqrt_fast(r[e], s2);
          slow = slow || s2;
        }
        if (__any_sync(kFull, slow)) {
#pragma unroll
          for (int e = 0; e < EPL; ++e) sr[e] = A::sqrt(r[e]);
        }
      }
#else
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        r[e] = A::rcp(xs[e]);
        sr[e] = A::sqrt(r[e]);
      }
#endif
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        const T cn = zc[e].c;
        // n = 0: powi gives exactly 1.0 and (c * 1.0) * sr == c * sr, so no select
        cur[e] = A::mul(A::mul(cn, powi_rt_bounded(r[e], n[e], bits)), sr[e]);
        if (wr[e]) dst[e][n[e]] = cur[e];
        tx[e] = A::add(xs[e], xs[e]);
      }
      // recursion steps m = wmax-1 .. 0: enter the unrolled chain once through
      // a jump table (wmax is warp-uniform) instead of testing every step
      // one predicate per element and step: elements that are not written
      // here (deferred, padding) take no steps (their cur is never used)
      int neff[EPL];
#pragma unroll
      for (int e = 0; e < EPL; ++e) neff[e] = wr[e] ? n[e] : 0;
#define BOYS_STEP(M)                                                       \
  if ((M) < NB) {                                                           \
    _Pragma("unroll") for (int e = 0; e < EPL; ++e) {                       \
      const T nx = A::mul(A::fma(tx[e], cur[e], t[e]), rinv<T>((M) < NB ? (M) : 0)); \
      const bool on = (M) < neff[e];                                        \
      pmov(on, cur[e], nx);                                                 \
      psts(on, dst[e] + (M), cur[e]);                                       \
    }                                                                       \
  }
      switch (wmax) {
        case 16: BOYS_STEP(15) [[fallthrough]];
        case 15: BOYS_STEP(14) [[fallthrough]];
        case 14: BOYS_STEP(13) [[fallthrough]];
        case 13: BOYS_STEP(12) [[fallthrough]];
        case 12: BOYS_STEP(11) [[fallthrough]];
        case 11: BOYS_STEP(10) [[fallthrough]];
        case 10: BOYS_STEP(9) [[fallthrough]];
        case 9: BOYS_STEP(8) [[fallthrough]];
        case 8: BOYS_STEP(7) [[fallthrough]];
        case 7: BOYS_STEP(6) [[fallthrough]];
        case 6: BOYS_STEP(5) [[fallthrough]];
        case 5: BOYS_STEP(4) [[fallthrough]];
        case 4: BOYS_STEP(3) [[fallthrough]];
        case 3: BOYS_STEP(2) [[fallthrough]];
        case 2: BOYS_STEP(1) [[fallthrough]];
        case 1: BOYS_STEP(0) [[fallthrough]];
        default: break;
      }
#undef BOYS_STEP
      static_assert(NB <= 16, "extend the recursion jump table");
      if (!kDeferUp<T>) {
        bool up[EPL], anyup = false;
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
          up[e] = wr[e] && xs[e] > zc[e].x_up;   // NaN (invalid) compares false
          anyup = anyup || up[e];
        }
        if (__any_sync(kFull, anyup)) {
#pragma unroll
          for (int e = 0; e < EPL; ++e) {
            const T rx = A::rcp(xs[e]);
            T f = up_first(xs[e]);
            if (up[e]) dst[e][0] = f;
#pragma unroll
            for (int m = 0; m < NB; ++m) {
              if (m >= wmax) break;
              f = up_next(f, m, rx);
              if (up[e] && m + 1 <= n[e]) dst[e][m + 1] = f;
            }
          }
        }
      }
    }
    __syncwarp();
    // the chunk's output range [base, base + cnt): scalar head/tail to reach
    // 16-byte alignment, one bulk async copy (TMA engine) for the body.
    // Deferred elements' slots go out stale and are rewritten by the drain.
    {
      const int ncnt = (int)cnt;
      const int head = ((Q - shift) & (Q - 1)) < ncnt ? ((Q - shift) & (Q - 1)) : ncnt;
      const int body = ((ncnt - head) / Q) * Q;
      const int tail0 = head + body;
      if (lane < head) __stcs(out + base + lane, W.stage[shift + lane]);
      if (lane < ncnt - tail0) __stcs(out + base + tail0 + lane, W.stage[shift + tail0 + lane]);
      if (body > 0) {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) bulk_store(out + base + head, W.stage + shift + head, body * sizeof(T));
      }
    }
    while (qn >= 32) ragged_drain<T, NB>(W, rows, qn, lane, out);
  }
  while (qn > 0) ragged_drain<T, NB>(W, rows, qn, lane, out);
  if (lane == 0) bulk_wait_all();
}

// (A block-window ragged variant -- 1024-element windows counting-sorted into
// order buckets, one compile-time-order tail per warp task -- measured slower
// than the warp chunks for both dtypes (f64 2.59 vs 1.92 ms, f32 1.19 vs
// 1.00 ms) and was removed; it is in the history up to commit 50d605b.)

// ---------------------------------------------------------------------------
// split kernel (eval_with_split): F_m for m <= nbar equals a
// dense order-nbar evaluation, F_m for m > nbar a dense order-n evaluation.
// ---------------------------------------------------------------------------
template <typename T, int n, bool AOS, int NBUF>
__global__ void __launch_bounds__(kThreads, AOS ? 4 : 1)
split_kernel(const T* __restrict__ X, int64_t N, int nbar, T* __restrict__ out,
             int64_t* __restrict__ dom, bool bulk_ok) {
  constexpr int W = n + 1;
  constexpr int TILE_ELEMS = kThreads * W;
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
      T* row = buf + tid * W;
      eval_point_stream<T, n>(x, ok, [&](int m, T v) { if (m > nbar) row[m] = v; });
      eval_point_uniform<T, n>(x, ok, nbar, ConstRows<T>{}, [&](int m, T v) { if (m <= nbar) row[m] = v; });
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
    } else {
      T* o = out + i;
      eval_point_stream<T, n>(x, ok, [&](int m, T v) {
        if (in && m > nbar) __stcs(o + (int64_t)m * N, v);
      });
      eval_point_uniform<T, n>(x, ok, nbar, ConstRows<T>{}, [&](int m, T v) {
        if (in && m <= nbar) __stcs(o + (int64_t)m * N, v);
      });
    }
  }
  if (AOS && tid == 0) bulk_wait_all();
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

// Persistent grid: SMs x resident blocks (measured better than one block per
// tile even for the 2^20-point config: block launch overhead dominates there).
// Opt a kernel in to more than 48 KB of dynamic shared memory on the current
// device (the attribute is per device; `mask` remembers which devices are done).
template <typename K>
static boys_status opt_in_smem(K kernel, int smem, std::atomic<uint64_t>& mask) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e);
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (mask.load(std::memory_order_acquire) & bit) return BOYS_OK;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return cuda_status(e);
  mask.fetch_or(bit, std::memory_order_acq_rel);
  return BOYS_OK;
}

// The occupancy query is cached per (kernel, shared-memory size): it is a
// host-side call that would otherwise sit on every launch's critical path.
template <typename K>
static int blocks_for(K kernel, size_t smem, int64_t ntiles, int threads = kThreads) {
  static thread_local struct { const void* k; size_t smem; int occ; } cache[8] = {};
  const void* key = reinterpret_cast<const void*>(kernel);
  int occ = 0;
  for (auto& c : cache)
    if (c.k == key && c.smem == smem) { occ = c.occ; break; }
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem);
    if (occ < 1) occ = 1;
    for (auto& c : cache)
      if (!c.k) { c = {key, smem, occ}; break; }
  }
  int64_t b = (int64_t)sm_count() * occ;
  if (ntiles < b) b = ntiles;
  return (int)(b < 1 ? 1 : b);
}

// Tuning knobs (read once; defaults = measured best on B200):
//   BOYS_AOS_NBUF  AoS staging depth per block (1 or 2)
//   BOYS_AOS_MINB  AoS resident-block target handed to __launch_bounds__ (4 or 6)
static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}
static int aos_nbuf() {
  static int v = env_int("BOYS_AOS_NBUF", 2) == 1 ? 1 : 2;
  return v;
}
static int soa_tma() {   // BOYS_SOA_TMA=1: SoA rows leave as bulk copies
  static int v = env_int("BOYS_SOA_TMA", 0);
  return v;
}
static int grid_tiles() {
  static int v = env_int("BOYS_GRID_TILES", 0);
  return v;
}
static int soa_small_minb() {   // BOYS_SOA0_MINB: 8 (default) or 6 for n <= 1
  static int v = env_int("BOYS_SOA0_MINB", 8) == 6 ? 6 : 8;
  return v;
}
static int soa_pair() {   // BOYS_SOA_PAIR=1: two adjacent points per thread (SoA)
  static int v = env_int("BOYS_SOA_PAIR", 1);
  return v;
}
// Grid for the paired SoA kernel (BOYS_PAIR_GRID: 0 = rule below, 1 = per
// tile, 2 = persistent).  Same-box sweeps (tools/ab/ab33.sh, 2^24 points):
// one block per 512-point tile wins for every f64 order (n=8: 230 vs 266 us,
// n=12: 314 vs 371 us) and for f32 n >= 6 (n=8: 112 vs 132 us); persistent
// for f32 n < 6 (n=4: 82 vs 90 us).
static bool soa_pair_per_tile(bool f64, int n) {
  static int v = env_int("BOYS_PAIR_GRID", 0);
  if (v) return v == 1;
  return f64 || n >= 6;
}
// Ragged grid = resident blocks x this (BOYS_RAGGED_GRID_MULT overrides).
// Same-box sweep (tools/ab/ab35.sh, cfg4): f64 best persistent (x1: 1.90 ms;
// x2 1.90, x4 1.91, x16 1.98); f32 best x4 (0.984 vs 1.007 ms at x1).
static int ragged_grid_mult(bool f64) {
  static int v = env_int("BOYS_RAGGED_GRID_MULT", 0);
  if (v >= 1) return v;
  return f64 ? 1 : 4;
}
static int pdl() {   // BOYS_PDL=0: plain stream-serialised launches (A/B)
  static int v = env_int("BOYS_PDL", 1);
  return v;
}
static int aos_minb() {
  static int v = env_int("BOYS_AOS_MINB", 4) == 6 ? 6 : 4;
  return v;
}

template <typename T, int n, bool AOS, int NBUF, int MINB>
static boys_status launch_dense_k(const T* x, int64_t N, T* out, T* expx, int64_t* dom,
                                  int64_t base, cudaStream_t s) {
  auto k = dense_kernel<T, n, AOS, NBUF, MINB>;
  // SoA bulk rows need every row start 16-byte aligned: N * sizeof(T) % 16 == 0
  const bool soa_bulk = !AOS && soa_tma() && (N * (int64_t)sizeof(T)) % 16 == 0 &&
                        (reinterpret_cast<uintptr_t>(out) % 16) == 0;
  size_t smem = (AOS || soa_bulk) ? (size_t)NBUF * kThreads * (n + 1) * sizeof(T) : 0;
  // the dynamic-smem opt-in is per function *per device*: remember each device
  static std::atomic<uint64_t> attr_mask{0};
  {
    const int smem_max = (int)((size_t)NBUF * kThreads * (n + 1) * sizeof(T));
    boys_status st = opt_in_smem(k, smem_max, attr_mask);
    if (st != BOYS_OK) return st;
  }
  int64_t ntiles = (N + kThreads - 1) / kThreads;
  bool bulk_ok = (reinterpret_cast<uintptr_t>(out) % 16) == 0;
  // Grid: persistent (SMs x resident blocks) or one block per tile, chosen
  // by same-box measurement (tools/ab/ab29.sh, ab30.sh; graph-replayed
  // streams at 2^20..2^24 points): one block per tile wins for f64 SoA at
  // n <= 5 and n >= 11 (n=0: 143 vs 154 us, n=16: 398 vs 471 us at 2^24),
  // persistent for f64 SoA n = 6..10 (n=8: 265 vs 282 us), for f32 SoA and for
  // AoS (whose double-buffered bulk stores need the loop).  BOYS_GRID_TILES=1/2
  // forces one or the other.
  int grid = blocks_for(k, smem, ntiles);
  const int gt = grid_tiles();
  const bool per_tile = gt == 1 || (gt == 0 && !AOS && !soa_bulk && sizeof(T) == 8 &&
                                    (n <= 5 || n >= 11));
  if (per_tile && ntiles <= (int64_t)1 << 30) grid = (int)ntiles;
  if (pdl()) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, x, N, out, expx, dom, base, bulk_ok, soa_bulk);
    if (e != cudaSuccess) return cuda_status(e);
  } else {
    k<<<grid, kThreads, smem, s>>>(x, N, out, expx, dom, base, bulk_ok, soa_bulk);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_status(cudaGetLastError());
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <typename T, int n>
static boys_status launch_soa_pair(const T* x, int64_t N, T* out, T* expx, int64_t* dom,
                                   int64_t base, cudaStream_t s) {
  constexpr int MINB = n <= 1 ? BOYS_PAIR_MINB_SMALL : BOYS_SOA_MINB;   // two chains: 8 blocks would spill at n = 0
  auto k = dense_soa_pair_kernel<T, n, MINB>;
  const int64_t ntiles = (N + 2 * kThreads - 1) / (2 * kThreads);
  int grid = blocks_for(k, 0, ntiles);
  const int gt = grid_tiles();
  if ((gt == 1 || (gt == 0 && soa_pair_per_tile(sizeof(T) == 8, n))) && ntiles <= ((int64_t)1 << 30))
    grid = (int)ntiles;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl() ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, x, N, out, expx, dom, base);
  if (e != cudaSuccess) return cuda_status(e);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_status(cudaGetLastError());
}

template <typename T, int n, bool AOS>
static boys_status launch_dense_t(const T* x, int64_t N, T* out, T* expx, int64_t* dom,
                                  int64_t base, cudaStream_t s) {
  if constexpr (!AOS) {
    constexpr bool fits2 = 2 * kThreads * (n + 1) * sizeof(T) <= 80 * 1024;
    if (soa_tma()) return launch_dense_k<T, n, false, (fits2 ? 2 : 1), 4>(x, N, out, expx, dom, base, s);
    if constexpr (n <= 1) {          // small orders: register budget for 6 or 8 blocks/SM
      if (soa_small_minb() == 6) return launch_dense_k<T, n, false, 1, 6>(x, N, out, expx, dom, base, s);
    }
    if (soa_pair() && N % 2 == 0 && aligned16(x) && aligned16(out) && (!expx || aligned16(expx)))
      return launch_soa_pair<T, n>(x, N, out, expx, dom, base, s);
    return launch_dense_k<T, n, false, 1, (n <= 1 ? 8 : BOYS_SOA_MINB)>(x, N, out, expx, dom, base, s);
  } else {
    // double-buffer the AoS tile while two tiles fit in ~80 KB (n <= 18 in f64)
    constexpr bool fits2 = 2 * kThreads * (n + 1) * sizeof(T) <= 80 * 1024;
    if (fits2 && aos_nbuf() == 2)
      return launch_dense_k<T, n, true, (fits2 ? 2 : 1), 4>(x, N, out, expx, dom, base, s);
    if (aos_minb() == 6) return launch_dense_k<T, n, true, 1, 6>(x, N, out, expx, dom, base, s);
    return launch_dense_k<T, n, true, 1, 4>(x, N, out, expx, dom, base, s);
  }
}

template <typename T, int n>
static boys_status dispatch_dense_layout(const void* x, int64_t N, void* out, boys_layout lay,
                                         void* expx, int64_t* dom, int64_t base, cudaStream_t s) {
  // n = 0: [N][1] and [1][N] are the same bytes; the SoA kernel (no staging)
  // measured faster (f64 2^24: 143 vs 167 us)
  if (lay == BOYS_AOS && n > 0)
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
  constexpr bool fits2 = 2 * kThreads * (n + 1) * sizeof(T) <= 80 * 1024;
  constexpr int NBUF = (AOS && fits2) ? 2 : 1;
  auto k = split_kernel<T, n, AOS, NBUF>;
  const size_t smem = AOS ? (size_t)NBUF * kThreads * (n + 1) * sizeof(T) : 0;
  static std::atomic<uint64_t> attr_mask{0};
  if (AOS) {
    boys_status st = opt_in_smem(k, (int)smem, attr_mask);
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

static int ragged_epl() {   // BOYS_RAGGED_EPL=1: one element per lane (A/B)
  static int v = env_int("BOYS_RAGGED_EPL", 0);
  return v;
}

template <typename T, int NB, int EPL, int CPE, int MINB, int WT = kThreads>
static boys_status launch_chunks(const void* x, const uint8_t* nm, const int64_t* off, int64_t N,
                                 void* out, int64_t* dom, cudaStream_t s) {
  auto k = ragged_kernel<T, NB, EPL, CPE, MINB, WT>;
  const size_t smem = sizeof(RaggedSmem<T, NB, EPL, CPE, WT>);
  static std::atomic<uint64_t> attr_mask{0};
  boys_status st = opt_in_smem(k, (int)smem, attr_mask);
  if (st != BOYS_OK) return st;
  const int64_t nch = (N + 32 * EPL - 1) / (32 * EPL);
  const int64_t nblk = (nch + WT / 32 - 1) / (WT / 32);
  int64_t grid = blocks_for(k, smem, nblk, WT);
  grid *= ragged_grid_mult(sizeof(T) == 8);
  if (grid > nblk) grid = nblk;
  k<<<(int)grid, WT, smem, s>>>((const T*)x, nm, off, N, (T*)out, dom);
  return BOYS_OK;
}

template <typename T>
static boys_status launch_ragged(const void* x, const uint8_t* nm, const int64_t* off, int64_t N,
                                 void* out, int64_t* dom, cudaStream_t s) {
  // fast-path order bound; higher orders, up to the table maximum, take the
  // in-kernel per-element fallback path
  constexpr int NB = Tab<T>::MAX_ORDER < kRaggedFastOrders ? Tab<T>::MAX_ORDER : kRaggedFastOrders;
  {
    // (order-sorted warp super-chunks were measured slower: 2.90 / 3.79 ms vs 2.42)
    // elements per lane: measured best 3 (f64: 1.95 ms vs 2.27 / 1.97 / 2.05
    // for 1 / 2 / 4) and 4 (f32: 1.14 ms vs 1.26 / 1.16 / 1.36 for 2 / 3 / 6)
    constexpr int EPL = sizeof(T) == 8 ? 3 : 4;
    // (8 instead of 12 staged values per element, or a 3-blocks/SM register
    // bound, measured no better: 1.96 / 2.08 ms f64)
    // (f64, 2 elements per lane with 10 staged values each, 24 warps/SM:
    // 1.88 ms -- within 1%, but overflows to the slow path from order 10)
    // (128-thread blocks, also with a 96-register bound and 8 staged values per
    // element for 20 resident warps, measured slower: f64 1.84-2.36 vs 1.78 ms,
    // f32 0.94-1.00 vs 0.94 ms, tools/ab/ab39.sh)
    boys_status st = ragged_epl() == 1
                         ? launch_chunks<T, NB, 1, NB + 1, 0>(x, nm, off, N, out, dom, s)
                         : launch_chunks<T, NB, EPL, 12, 0>(x, nm, off, N, out, dom, s);
    if (st != BOYS_OK) return st;
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

// ragged host-buffer pipeline workspace (per device, grown on demand, reused)
struct RaggedPipe {
  int device = -1;
  size_t cap_x = 0, cap_n = 0, cap_off = 0, cap_out = 0, cap_dom = 0;
  void* dx[2] = {nullptr, nullptr};
  uint8_t* dn[2] = {nullptr, nullptr};
  int64_t* doff[2] = {nullptr, nullptr};
  void* dout[2] = {nullptr, nullptr};
  int64_t* ddom = nullptr;       // one first-bad index per chunk
  cudaStream_t st[2] = {nullptr, nullptr};
};
static std::vector<RaggedPipe> g_rpipes;

static cudaError_t grow(void** p, size_t& cap, size_t need) {
  if (need <= cap) return cudaSuccess;
  cudaFree(*p);
  *p = nullptr;
  cap = 0;
  cudaError_t e = cudaMalloc(p, need);
  if (e == cudaSuccess) cap = need;
  return e;
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

boys_status boys_eval_ragged_host(boys_dtype dtype, const void* x_host, const uint8_t* nmax_host,
                                  int64_t N, void* out_host, int64_t out_capacity,
                                  int64_t* first_bad) {
  if (dtype != BOYS_F64 && dtype != BOYS_F32) return BOYS_E_DTYPE;
  if (N < 0 || out_capacity < 0) return BOYS_E_ARG;
  if (first_bad) *first_bad = -1;
  if (N == 0) return BOYS_OK;
  if (!x_host || !nmax_host || !out_host) return BOYS_E_ARG;
  std::lock_guard<std::mutex> lk(g_pipe_mu);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e);
  RaggedPipe* p = nullptr;
  for (auto& q : g_rpipes)
    if (q.device == dev) { p = &q; break; }
  if (!p) {
    g_rpipes.emplace_back();
    p = &g_rpipes.back();
    p->device = dev;
    for (auto& st : p->st) {
      e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
      if (e != cudaSuccess) return cuda_status(e);
    }
  }
  const size_t es = dsize(dtype);
  const int64_t chunk = N < (int64_t(1) << 22) ? N : (int64_t(1) << 22);
  const int64_t nchunks = (N + chunk - 1) / chunk;
  // per-chunk domain slots; x/n/offsets buffers sized once for the chunk
  for (int k = 0; k < 2; ++k) {
    size_t cx = p->cap_x, cn = p->cap_n, co = p->cap_off;
    if ((e = grow(&p->dx[k], cx, chunk * es)) != cudaSuccess) return cuda_status(e);
    if ((e = grow((void**)&p->dn[k], cn, chunk)) != cudaSuccess) return cuda_status(e);
    if ((e = grow((void**)&p->doff[k], co, (chunk + 1) * sizeof(int64_t))) != cudaSuccess)
      return cuda_status(e);
    if (k == 1) { p->cap_x = cx; p->cap_n = cn; p->cap_off = co; }
  }
  if ((e = grow((void**)&p->ddom, p->cap_dom, nchunks * sizeof(int64_t))) != cudaSuccess)
    return cuda_status(e);
  e = cudaMemsetAsync(p->ddom, 0xff, nchunks * sizeof(int64_t), p->st[0]);
  if (e != cudaSuccess) return cuda_status(e);
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  cudaEventRecord(ev, p->st[0]);
  cudaStreamWaitEvent(p->st[1], ev, 0);
  const uint8_t* nh = nmax_host;
  int64_t base = 0;
  boys_status st = BOYS_OK;
  for (int64_t c = 0; c < nchunks && st == BOYS_OK; ++c) {
    const int k = (int)(c & 1);
    cudaStream_t s = p->st[k];
    const int64_t i0 = c * chunk;
    const int64_t cn = (N - i0) < chunk ? (N - i0) : chunk;
    // the chunk's output length (host pass over its orders, overlapped with
    // the device work already queued for earlier chunks)
    int64_t total = cn;
    for (int64_t i = 0; i < cn; ++i) total += nh[i0 + i];
    if (base + total > out_capacity) { st = BOYS_E_ARG; break; }
    if ((size_t)total * es > p->cap_out) {     // grow both output slots (rare)
      for (auto ss : p->st) cudaStreamSynchronize(ss);
      size_t need = (size_t)total * es + (size_t)total * es / 4;
      for (int q = 0; q < 2; ++q) {
        size_t cap = p->cap_out;
        if ((e = grow(&p->dout[q], cap, need)) != cudaSuccess) { st = cuda_status(e); break; }
        if (q == 1) p->cap_out = cap;
      }
      if (st != BOYS_OK) break;
    }
    e = cudaMemcpyAsync(p->dx[k], (const char*)x_host + i0 * es, cn * es, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(p->dn[k], nh + i0, cn, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) { st = cuda_status(e); break; }
    st = boys_ragged_offsets(p->dn[k], cn, p->doff[k], s);
    if (st != BOYS_OK) break;
    st = dtype == BOYS_F64
             ? launch_ragged<double>(p->dx[k], p->dn[k], p->doff[k], cn, p->dout[k], p->ddom + c, s)
             : launch_ragged<float>(p->dx[k], p->dn[k], p->doff[k], cn, p->dout[k], p->ddom + c, s);
    if (st != BOYS_OK) break;
    e = cudaMemcpyAsync((char*)out_host + base * es, p->dout[k], total * es, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) { st = cuda_status(e); break; }
    base += total;
  }
  for (auto s : p->st) {
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess && st == BOYS_OK) st = cuda_status(e);
  }
  cudaEventDestroy(ev);
  if (st != BOYS_OK) return st;
  std::vector<int64_t> dom(nchunks);
  e = cudaMemcpy(dom.data(), p->ddom, nchunks * sizeof(int64_t), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_status(e);
  for (int64_t c = 0; c < nchunks; ++c)
    if (dom[c] >= 0) {
      if (first_bad) *first_bad = c * chunk + dom[c];
      return BOYS_E_DOMAIN;
    }
  return BOYS_OK;
}

}  // extern "C"
