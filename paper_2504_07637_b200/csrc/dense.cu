// Dense kernels (one order for the whole batch): the multi-point SoA kernels
// (four / two adjacent points per thread), the paired AoS kernel, the one-point
// SoA / AoS kernel, and their launch rules.  Part of libboys.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <type_traits>

#include "boys_device.cuh"
#include "boys_launch.h"

namespace boys {

// Where the multi-point kernels take the branch-free correctly rounded
// div/sqrt/rcp (seed_multi_fast), by same-box order sweep at 2^24 (f64): the
// AoS register-row kernel (n=1: 0.1232 -> 0.1141 ms, n=2: 0.1365 -> 0.1248)
// and the SoA pair kernel from n = 11 (1-2% faster); not the SoA pair kernel
// at n = 4..8 (5-11% slower: cfg2 0.208 vs 0.221 ms) nor the AoS pair kernel
// (n=3..8: 2-12% slower) -- more registers where the kernel is HBM-bound.
template <typename T, int n> constexpr bool kFastVec = sizeof(T) == 8;
template <typename T, int n> constexpr bool kFastSoaPair = sizeof(T) == 8 && n >= 11;
// AoS register rows: the fast paths' fallbacks as volatile asm at n = 3 (f64
// 2^24 points: 0.154 vs 0.168 ms; n = 1, 2 measured no gain)
template <int n> constexpr bool kColdVec = n == 3;

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
  // pre-wait L2 prefetch (boys_device.cuh): f64 every order (2^24 points: 0 to
  // -1.6%), f32 where it measured faster (n = 9..11: -3 to -9%, n <= 7: 0 to
  // -2%; n = 8 and n >= 12 measured +1 to +3% and skip it)
  if constexpr (sizeof(T) == 8 || (n != 8 && n < 12)) prefetch_first_tile(X, N, TILE);
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
    eval_pair_stream<T, n, kFastSoaPair<T, n>>(
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

// SoA dense kernel, four adjacent points per thread (1024-point tiles): x as
// two 16-byte loads, every F_m row as two 16-byte streaming stores.  N % 4 == 0
// and 16-byte aligned buffers (host checks).  A/B variant for the FP64-bound
// small orders.
template <typename T, int n, int MINB, bool FAST>
__global__ void __launch_bounds__(kThreads, MINB)
dense_soa_quad_kernel(const T* __restrict__ X, int64_t N, T* __restrict__ out,
                      T* __restrict__ expx, int64_t* __restrict__ dom, int64_t index_base) {
  using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
  const int tid = threadIdx.x;
  constexpr int TILE = 4 * kThreads;
  const int64_t ntiles = (N + TILE - 1) / TILE;
  pdl_wait_and_release();
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i = tile * TILE + 4 * tid;     // N % 4 == 0 => all four in range iff i < N
    const bool in = i < N;
    T xv[4];
    bool ok[4];
    if (in) {
      const V2 a = __ldg(reinterpret_cast<const V2*>(X + i));
      const V2 b = __ldg(reinterpret_cast<const V2*>(X + i + 2));
      xv[0] = a.x; xv[1] = a.y; xv[2] = b.x; xv[3] = b.y;
    } else {
      xv[0] = xv[1] = xv[2] = xv[3] = T(0);
    }
    bool bad = false;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      ok[j] = valid_x(xv[j]) || !in;
      bad = bad || !ok[j];
    }
    if (__any_sync(kFull, bad)) {                  // rare: one vote per thread, not a branch per point
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (!ok[j]) flag_domain(dom, index_base + i + j);
    }
    T* o = out + i;
    T tv[4];
    eval_multi_stream<T, n, 4, FAST>(
        xv, ok, tv,
        [&](int m, const T (&v)[4]) {
          if (in) {
            V2 a, b;
            a.x = v[0]; a.y = v[1]; b.x = v[2]; b.y = v[3];
            __stcs(reinterpret_cast<V2*>(o + (int64_t)m * N), a);
            __stcs(reinterpret_cast<V2*>(o + (int64_t)m * N + 2), b);
          }
        },
        [&](int j, int m, T v) {
          if (in) __stcs(o + (int64_t)m * N + j, v);
        });
    if (expx && in) {
      V2 a, b;
      a.x = tv[0]; a.y = tv[1]; b.x = tv[2]; b.y = tv[3];
      __stcs(reinterpret_cast<V2*>(expx + i), a);
      __stcs(reinterpret_cast<V2*>(expx + i + 2), b);
    }
  }
}

// Four points of a thread at n = 0: domain check, F_0 and e^{-x} into
// registers (shared by the speculative kernel below and its cold re-run).
template <typename T>
__device__ __forceinline__ void quad0_eval(const T (&xv)[4], bool in, T (&fv)[4], T (&tv)[4],
                                           bool (&ok)[4], bool& any_bad) {
  bool bad = false;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    ok[j] = surely_valid_x(xv[j]);
    bad = bad || !ok[j];
  }
  any_bad = __any_sync(kFull, bad);
  if (any_bad) {                                   // rare
    bad = false;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      ok[j] = valid_x(xv[j]) || !in;
      bad = bad || !ok[j];
    }
    any_bad = __any_sync(kFull, bad);
  }
  eval_multi_stream<T, 0, 4, true, true, true>(
      xv, ok, tv,
      [&](int, const T (&v)[4]) {
#pragma unroll
        for (int j = 0; j < 4; ++j) fv[j] = v[j];
      },
      [&](int, int, T) {}, any_bad);
}

template <typename T>
__device__ __forceinline__ void quad0_store(const T (&fv)[4], const T (&tv)[4], const bool (&ok)[4],
                                            bool any_bad, bool in, int64_t i, T* __restrict__ out,
                                            T* __restrict__ expx, int64_t* __restrict__ dom,
                                            int64_t index_base) {
  using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
  if (any_bad) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (!ok[j]) flag_domain(dom, index_base + i + j);
  }
  if (in) {
    V2 a, b;
    a.x = fv[0]; a.y = fv[1]; b.x = fv[2]; b.y = fv[3];
    __stcs(reinterpret_cast<V2*>(out + i), a);
    __stcs(reinterpret_cast<V2*>(out + i + 2), b);
    if (expx) {
      a.x = tv[0]; a.y = tv[1]; b.x = tv[2]; b.y = tv[3];
      __stcs(reinterpret_cast<V2*>(expx + i), a);
      __stcs(reinterpret_cast<V2*>(expx + i + 2), b);
    }
  }
}

// n = 0 variant of the four-point SoA kernel that computes BEFORE waiting on
// the stream's previous grid: each block loads its x tile and evaluates F_0
// into registers while the previous grid's tail is still draining, then
// waits (griddepcontrol.wait: the previous grid has completed and its writes
// are visible), re-reads x past L1 and compares bit for bit.  Equal (x was not
// produced by the previous grid -- the usual case): the results are stored.
// Different: the tile is evaluated again, now after the wait.  Nothing
// is written and no domain flag is raised before the wait, so the launch stays
// stream-ordered for every buffer; the only early accesses are reads of x,
// whose values are confirmed afterwards.  One row of results (8 registers) is
// held across the wait, which is why only n = 0 does this.  A stream of
// 2^20-point launches keeps the FP64 pipe busy across launch boundaries.
template <typename T, int MINB, bool EXPX>
__global__ void __launch_bounds__(kThreads, MINB)
dense_soa_quad0_spec_kernel(const T* __restrict__ X, int64_t N, T* __restrict__ out,
                            T* __restrict__ expx_arg, int64_t* __restrict__ dom,
                            int64_t index_base, int ahead) {
  T* __restrict__ expx = EXPX ? expx_arg : nullptr;  // without it the e^{-x} row is dead code
  using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
  const int tid = threadIdx.x;
  constexpr int TILE = 4 * kThreads;
  const int64_t ntiles = (N + TILE - 1) / TILE;
  // dependents wait for this grid's completion themselves before they store
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  bool waited = false;                             // block-uniform
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i = tile * TILE + 4 * tid;     // N % 4 == 0 => all four in range iff i < N
    const bool in = i < N;
    V2 xa, xb;
    xa.x = xa.y = xb.x = xb.y = T(0);
    if (in) {
      xa = __ldcg(reinterpret_cast<const V2*>(X + i));
      xb = __ldcg(reinterpret_cast<const V2*>(X + i + 2));
    }
#ifndef BOYS_AB_NOAHEAD
    // L2 prefetch for the block that takes this one's place (`ahead` = resident
    // blocks of the grid): the next wave starts all at once when this one
    // leaves, and would otherwise open with a DRAM round trip
    if (tile + ahead < ntiles) {
      constexpr int PER = 32 / (int)sizeof(T);
      if (tid * PER < TILE) prefetch_l2(X + (tile + ahead) * TILE + tid * PER);
    }
#endif
    const T xv[4] = {xa.x, xa.y, xb.x, xb.y};
    T fv[4], tv[4];
    bool ok[4], any_bad;
    quad0_eval<T>(xv, in, fv, tv, ok, any_bad);
    if (!waited) {
      asm volatile("griddepcontrol.wait;\n" ::: "memory");
      waited = true;
      const V2 pa = xa, pb = xb;
      V2 ya = pa, yb = pb;
      if (in) {
        ya = __ldcg(reinterpret_cast<const V2*>(X + i));
        yb = __ldcg(reinterpret_cast<const V2*>(X + i + 2));
      }
      const bool diff = !same_bits(ya.x, pa.x) || !same_bits(ya.y, pa.y) ||
                        !same_bits(yb.x, pb.x) || !same_bits(yb.y, pb.y);
      if (__any_sync(kFull, diff)) {               // speculation failed: this tile again, now after the wait
        tile -= gridDim.x;
        continue;
      }
    }
    quad0_store<T>(fv, tv, ok, any_bad, in, i, out, expx, dom, index_base);
  }
  if (!waited) asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

// AoS dense kernel for rows of 2 or 4 values (n = 1, 3): P adjacent points per
// thread, each point's row kept in registers and written straight to global
// memory as 16-byte vectors (the thread's P rows are contiguous), no shared
// staging.  N % P == 0 and 16-byte aligned buffers (host checks).
template <typename T, int n, int P, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
dense_aos_vec_kernel(const T* __restrict__ X, int64_t N, T* __restrict__ out,
                     T* __restrict__ expx, int64_t* __restrict__ dom, int64_t index_base) {
  using V2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
  constexpr int W = n + 1;
  static_assert((P * W) % 2 == 0 && P % 2 == 0, "P rows of W values: whole 16-byte vectors");
  const int tid = threadIdx.x;
  constexpr int TILE = P * kThreads;
  const int64_t ntiles = (N + TILE - 1) / TILE;
  pdl_wait_and_release();
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i = tile * TILE + P * tid;     // N % P == 0 => all P in range iff i < N
    const bool in = i < N;
    T xv[P], tv[P], row[P][W];
    bool ok[P];
#pragma unroll
    for (int j = 0; j < P; j += 2) {
      V2 a;
      if (in) a = __ldg(reinterpret_cast<const V2*>(X + i + j));
      else { a.x = T(0); a.y = T(0); }
      xv[j] = a.x;
      xv[j + 1] = a.y;
    }
#pragma unroll
    for (int j = 0; j < P; ++j) {
      ok[j] = valid_x(xv[j]);
      if (in && !ok[j]) flag_domain(dom, index_base + i + j);
      ok[j] = ok[j] || !in;
    }
    eval_multi_stream<T, n, P, kFastVec<T, n>, false, kColdVec<n>>(
        xv, ok, tv,
        [&](int m, const T (&v)[P]) {
#pragma unroll
          for (int j = 0; j < P; ++j) row[j][m] = v[j];
        },
        [&](int j, int m, T v) { row[j][m] = v; });
    if (in) {
      // the thread's P rows are P*W contiguous values starting at a 16-byte
      // boundary (i is a multiple of P, P even): whole 16-byte vectors
      V2* o = reinterpret_cast<V2*>(out + i * W);
#pragma unroll
      for (int f = 0; f < P * W; f += 2) {
        V2 v;
        v.x = row[f / W][f % W];
        v.y = row[(f + 1) / W][(f + 1) % W];
        __stcs(o + f / 2, v);
      }
      if (expx) {
#pragma unroll
        for (int j = 0; j < P; j += 2) {
          V2 v;
          v.x = tv[j];
          v.y = tv[j + 1];
          __stcs(reinterpret_cast<V2*>(expx + i + j), v);
        }
      }
    }
  }
}

// AoS dense kernel, two points per thread (i0 + tid and i0 + 256 + tid of a
// 512-point tile), evaluated in lockstep (eval_pair_stream); the [512][n+1]
// tile is staged in shared memory and leaves as one bulk copy, NBUF-deep.
// A/B variant for orders whose double-buffered tile still fits 2 blocks/SM.
template <typename T, int n, int NBUF, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
dense_aos_pair_kernel(const T* __restrict__ X, int64_t N, T* __restrict__ out,
                      T* __restrict__ expx, int64_t* __restrict__ dom, int64_t index_base,
                      bool bulk_ok) {
  constexpr int W = n + 1, WS = RowStride<W>::value;
  constexpr int TILE = 2 * kThreads;
  constexpr int TILE_ELEMS = TILE * WS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* sbase = reinterpret_cast<T*>(smem_raw);
  const int tid = threadIdx.x;
  const int64_t ntiles = (N + TILE - 1) / TILE;
  pdl_wait_and_release();
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int64_t i0 = tile * TILE;
    const int64_t ia = i0 + tid, ib = i0 + kThreads + tid;
    const bool ina = ia < N, inb = ib < N;
    const T xa = ina ? ldg_nc(X + ia) : T(0);
    const T xb = inb ? ldg_nc(X + ib) : T(0);
    bool oka = valid_x(xa), okb = valid_x(xb);
    if (ina && !oka) flag_domain(dom, index_base + ia);
    if (inb && !okb) flag_domain(dom, index_base + ib);
    oka = oka || !ina;
    okb = okb || !inb;
    T* buf = sbase + (it % NBUF) * TILE_ELEMS;
    if (tid == 0) bulk_wait_read<NBUF - 1>();
    __syncthreads();
    T* ra = buf + tid * WS;
    T* rb = buf + (kThreads + tid) * WS;
    T ta, tb;
    eval_pair_stream<T, n>(
        xa, xb, oka, okb, ta, tb,
        [&](int m, T a, T b) { ra[m] = a; rb[m] = b; },
        [&](int j, int m, T v) { (j == 0 ? ra : rb)[m] = v; });
    if (expx) {
      if (ina) __stcs(expx + ia, ta);
      if (inb) __stcs(expx + ib, tb);
    }
    const int64_t cnt = (N - i0) < TILE ? (N - i0) : TILE;
    if (!RowStride<W>::padded && bulk_ok && cnt == TILE) {
      fence_proxy_async_smem();
      __syncthreads();
      if (tid == 0) bulk_store(out + i0 * W, buf, TILE_ELEMS * sizeof(T));
    } else {
      __syncthreads();
      copy_out_rows<T, W, WS>(out + i0 * W, buf, cnt, tid, kThreads);
    }
  }
  if (tid == 0) bulk_wait_all();
}

// ---------------------------------------------------------------------------
// dense kernel
// ---------------------------------------------------------------------------
template <typename T, int n, bool AOS, int NBUF, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
dense_kernel(const T* __restrict__ X, int64_t N, T* __restrict__ out, T* __restrict__ expx,
             int64_t* __restrict__ dom, int64_t index_base, bool bulk_ok) {
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
    // (loading the next tile's x one iteration ahead measured slower:
    // SoA 77% vs 84%, AoS 86% vs 94% of HBM; an L2 prefetch of it instead:
    // cfg3 1.688 vs 1.572 ms)
    const T x = in ? ldg_nc(X + i) : T(0);
    bool ok = valid_x(x);
    if (in && !ok) flag_domain(dom, index_base + i);
    ok = ok || !in;   // tail lanes evaluate x = 0 quietly
    if constexpr (!AOS) {
      T* o = out + i;
      T t = eval_point_stream<T, n>(x, ok, [&](int m, T v) {
        if (in) __stcs(o + (int64_t)m * N, v);
      });
      if (expx && in) __stcs(expx + i, t);
    } else {
      T* buf = sbase + (it % NBUF) * TILE_ELEMS;
      // the slot went to the bulk engine NBUF tiles ago: wait until it was read
      if (tid == 0) bulk_wait_read<NBUF - 1>();
      __syncthreads();
      T* row = buf + tid * WS;
      T t = eval_point_stream<T, n>(x, ok, [&](int m, T v) { row[m] = v; });
      if (expx && in) __stcs(expx + i, t);
      const int64_t cnt = (N - i0) < kThreads ? (N - i0) : kThreads;
      if (!RowStride<W>::padded && bulk_ok && cnt == kThreads) {
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) bulk_store(out + i0 * W, buf, TILE_ELEMS * sizeof(T));
      } else {
        __syncthreads();
        copy_out_rows<T, W, WS>(out + i0 * W, buf, cnt, tid, kThreads);
      }
    }
  }
  if (AOS && tid == 0) bulk_wait_all();
}

// ---------------------------------------------------------------------------
// launches.  Every dense kernel is launched with programmatic stream
// serialization (PDL): its blocks wait for the previous grid at entry
// (pdl_wait_and_release), so only the launch and prologue overlap the
// previous kernel's tail.  Kernel and grid choices below are fixed rules, each
// chosen by same-box B200 measurement (DESIGN.md section 6 records the A/B
// numbers; the losing variants were removed).
// ---------------------------------------------------------------------------
template <typename K, typename... Args>
static boys_status launch_pdl(K kernel, int grid, size_t smem, cudaStream_t s, Args... args) {
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
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, args...);
  if (e != cudaSuccess) return cuda_status(e);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_status(cudaGetLastError());
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
// one block per tile (falls back to a persistent grid past 2^30 tiles)
template <typename K>
static int per_tile_grid(K kernel, size_t smem, int64_t ntiles) {
  return ntiles <= ((int64_t)1 << 30) ? (int)ntiles : blocks_for(kernel, smem, ntiles);
}

// one-point kernel: SoA fallback (odd N / unaligned buffers) and AoS rows that
// do not fit the paired / register-row kernels
template <typename T, int n, bool AOS, int NBUF, int MINB>
static boys_status launch_dense_k(const T* x, int64_t N, T* out, T* expx, int64_t* dom,
                                  int64_t base, cudaStream_t s) {
  auto k = dense_kernel<T, n, AOS, NBUF, MINB>;
  const size_t smem = AOS ? (size_t)NBUF * kThreads * RowStride<n + 1>::value * sizeof(T) : 0;
  // the dynamic-smem opt-in is per function *per device*: remember each device
  static std::atomic<uint64_t> attr_mask{0};
  if (AOS) {
    boys_status st = opt_in_smem(k, (int)smem, attr_mask);
    if (st != BOYS_OK) return st;
  }
  const int64_t ntiles = (N + kThreads - 1) / kThreads;
  const bool bulk_ok = aligned16(out);
  // one block per tile for f64 SoA at n <= 5 and n >= 11 (n=0: 143 vs 154 us,
  // n=16: 398 vs 471 us at 2^24); persistent otherwise (f64 SoA n=6..10: n=8
  // 265 vs 282 us; f32 SoA; AoS, whose double-buffered bulk stores need the loop)
  const bool per_tile = !AOS && sizeof(T) == 8 && (n <= 5 || n >= 11);
  const int grid = per_tile ? per_tile_grid(k, smem, ntiles) : blocks_for(k, smem, ntiles);
  return launch_pdl(k, grid, smem, s, x, N, out, expx, dom, base, bulk_ok);
}

// SoA, two adjacent points per thread: one block per 512-point tile for every
// f64 order (n=8: 230 vs 266 us, n=12: 314 vs 371 us at 2^24) and f32 n >= 6;
// persistent for f32 n < 6 (n=4: 82 vs 90 us)
template <typename T, int n>
static boys_status launch_soa_pair(const T* x, int64_t N, T* out, T* expx, int64_t* dom,
                                   int64_t base, cudaStream_t s) {
  // resident-block targets: two chains would spill at 8 blocks for n <= 1
  // (5: 47 registers, cfg1 9.27 us vs 9.50 / 9.71 / 9.65 / 9.75 for 6 / 4 / 3 / 8)
  constexpr int MINB = n <= 1 ? 5 : 4;
  auto k = dense_soa_pair_kernel<T, n, MINB>;
  const int64_t ntiles = (N + 2 * kThreads - 1) / (2 * kThreads);
  const bool per_tile = sizeof(T) == 8 || n >= 6;
  const int grid = per_tile ? per_tile_grid(k, 0, ntiles) : blocks_for(k, 0, ntiles);
  return launch_pdl(k, grid, 0, s, x, N, out, expx, dom, base);
}

// SoA, four adjacent points per thread (n <= 5: f64 2^24 n=0 113 vs 123 us,
// n=1 122 vs 135, n=3 152 vs 167; f32 n <= 2 9-13% faster), one block per
// 1024-point tile (persistent: cfg1 10.8 vs 9.25 us), 4 resident blocks (59-64
// registers; 3 / 2: slower), branch-free correctly rounded div/sqrt/rcp.
template <typename T, int n>
static boys_status launch_soa_quad(const T* x, int64_t N, T* out, T* expx, int64_t* dom,
                                   int64_t base, cudaStream_t s) {
  const int64_t ntiles = (N + 4 * kThreads - 1) / (4 * kThreads);
  // n = 0, up to 2^22 points: the speculative kernel (a stream of 2^20-point
  // launches: 6.9 vs 7.7 us per launch; three resident blocks, no spills: four
  // measured 1.8% slower).  Larger launches gain nothing at their boundaries
  // and pay the re-read (2^26 points: +1.2-2.5%), so they keep the plain kernel.
  if constexpr (n == 0) {
    if (N <= (int64_t(1) << 22)) {
      if (expx) {
        auto k0 = dense_soa_quad0_spec_kernel<T, 3, true>;
        const int ahead = blocks_for(k0, 0, int64_t(1) << 40);     // resident blocks
        return launch_pdl(k0, per_tile_grid(k0, 0, ntiles), 0, s, x, N, out, expx, dom, base, ahead);
      }
      auto k0 = dense_soa_quad0_spec_kernel<T, 3, false>;
      const int ahead = blocks_for(k0, 0, int64_t(1) << 40);
      return launch_pdl(k0, per_tile_grid(k0, 0, ntiles), 0, s, x, N, out, expx, dom, base, ahead);
    }
  }
  auto k = dense_soa_quad_kernel<T, n, 4, true>;
  return launch_pdl(k, per_tile_grid(k, 0, ntiles), 0, s, x, N, out, expx, dom, base);
}

// AoS rows of 2..4 values kept in registers, P points per thread, direct
// 16-byte stores, one block per tile
template <typename T, int n, int P>
static boys_status launch_aos_vec(const T* x, int64_t N, T* out, T* expx, int64_t* dom,
                                  int64_t base, cudaStream_t s) {
  auto k = dense_aos_vec_kernel<T, n, P, 4>;
  const int64_t ntiles = (N + P * kThreads - 1) / (P * kThreads);
  return launch_pdl(k, per_tile_grid(k, 0, ntiles), 0, s, x, N, out, expx, dom, base);
}

// AoS, two points per thread with the [512][n+1] tile staged and bulk-stored
template <typename T, int n>
static boys_status launch_aos_pair(const T* x, int64_t N, T* out, T* expx, int64_t* dom,
                                   int64_t base, cudaStream_t s) {
  constexpr size_t tile_bytes = (size_t)2 * kThreads * RowStride<n + 1>::value * sizeof(T);
  constexpr int NBUF = (2 * tile_bytes <= 110 * 1024 && !RowStride<n + 1>::padded) ? 2 : 1;
  constexpr int MINB = NBUF * tile_bytes <= 72 * 1024 ? 3 : 2;
  auto k = dense_aos_pair_kernel<T, n, NBUF, MINB>;
  const size_t smem = NBUF * tile_bytes;
  static std::atomic<uint64_t> attr_mask{0};
  boys_status st = opt_in_smem(k, (int)smem, attr_mask);
  if (st != BOYS_OK) return st;
  const int64_t ntiles = (N + 2 * kThreads - 1) / (2 * kThreads);
  return launch_pdl(k, blocks_for(k, smem, ntiles), smem, s, x, N, out, expx, dom, base,
                    aligned16(out));
}

template <typename T, int n, bool AOS>
static boys_status launch_dense_t(const T* x, int64_t N, T* out, T* expx, int64_t* dom,
                                  int64_t base, cudaStream_t s) {
  const bool al = aligned16(x) && aligned16(out) && (!expx || aligned16(expx));
  if constexpr (!AOS) {
    // four points per thread (with the branch-free CR fast paths) up to n = 5:
    // same-box sweep at 2^24, f64 n=4 0.1646 -> 0.1393 ms, n=5 0.1748 -> 0.1586
    // vs the pair kernel; f32 n=4, 5 1-2% faster; slower from n = 6 (f64 n=7
    // +20%: registers where the order is HBM-bound)
    if constexpr (n <= 5) {
      if (N % 4 == 0 && al) return launch_soa_quad<T, n>(x, N, out, expx, dom, base, s);
    }
    if (N % 2 == 0 && al) return launch_soa_pair<T, n>(x, N, out, expx, dom, base, s);
    return launch_dense_k<T, n, false, 1, (n <= 1 ? 8 : 4)>(x, N, out, expx, dom, base, s);
  } else {
    if constexpr (n >= 1 && n <= 3) {
      // register rows + direct 16-byte stores for n = 1..3 (2^24: n=1 f64 128.6
      // vs 158.2 us, f32 63.4 vs 91.2; n=2 f64 149.2 vs 168.1, f32 82.9 vs
      // 96.2; f32 n=3 88.1 vs 97.8; f64 n=3, with the CR fast paths, 0.1683 vs
      // 0.1715 ms for the paired staged kernel; f64 n=4, 5 slower: +3%, +25%)
      constexpr int P = (n == 1 || (n == 2 && sizeof(T) == 8)) ? 4 : 2;
      constexpr bool use = true;
      if (use && N % P == 0 && al) return launch_aos_vec<T, n, P>(x, N, out, expx, dom, base, s);
    }
    // paired AoS where the double-buffered 512-point tile allows 3 blocks/SM
    // (f64 n <= 8, every f32 order: f64 n=2 168 vs 196 us, n=8 241 vs 248;
    // f32 n=8 116 vs 144, n=16 197 vs 217; slower for f64 n >= 10)
    if constexpr (2 * 2 * kThreads * (n + 1) * sizeof(T) <= 72 * 1024)
      return launch_aos_pair<T, n>(x, N, out, expx, dom, base, s);
    // one point per thread, the AoS tile double-buffered while two tiles fit
    // in ~80 KB (f64 n <= 18)
    // (padded rows leave through synchronous thread stores: one buffer)
    constexpr bool fits2 = 2 * kThreads * (n + 1) * sizeof(T) <= 80 * 1024 &&
                           !RowStride<n + 1>::padded;
    return launch_dense_k<T, n, true, (fits2 ? 2 : 1), 4>(x, N, out, expx, dom, base, s);
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

boys_status eval_dense_base(boys_dtype dtype, int n_max, const void* x, int64_t N,
                            void* out, boys_layout lay, void* expx, int64_t* dom,
                            int64_t base, cudaStream_t s) {
  if (dtype == BOYS_F64) return dispatch_dense<double>(n_max, x, N, out, lay, expx, dom, base, s);
  return dispatch_dense<float>(n_max, x, N, out, lay, expx, dom, base, s);
}

}  // namespace boys
