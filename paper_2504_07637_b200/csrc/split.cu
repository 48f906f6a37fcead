// eval_with_split: two seeds, two recursions.  Part of libboys.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <type_traits>

#include "boys_device.cuh"
#include "boys_launch.h"

namespace boys {

#ifndef BOYS_SPLIT_SOA_MINB
#define BOYS_SPLIT_SOA_MINB 3   // SoA split: 3 resident blocks (80 regs); unbounded (134 regs, 1 block) was 2x slower (ab55)
#endif

// ---------------------------------------------------------------------------
// split kernel (eval_with_split): F_m for m <= nbar equals a
// dense order-nbar evaluation, F_m for m > nbar a dense order-n evaluation.
// ---------------------------------------------------------------------------
template <typename T, int n, bool AOS, int NBUF>
__global__ void __launch_bounds__(kThreads, AOS ? 4 : BOYS_SPLIT_SOA_MINB)
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

boys_status eval_split_base(boys_dtype dtype, int n, int n_bar, const void* x, int64_t N,
                            void* out, boys_layout lay, int64_t* dom, cudaStream_t s) {
  if (dtype == BOYS_F64) return dispatch_split<double>(n, n_bar, x, N, out, lay, dom, s);
  return dispatch_split<float>(n, n_bar, x, N, out, lay, dom, s);
}

}  // namespace boys
