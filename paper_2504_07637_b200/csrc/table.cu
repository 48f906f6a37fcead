// Run-time coefficient tables (eval_batch / eval_with_split
// take a KernelTable, loaded from the coefficient dataset).  The compiled-in
// __constant__ tables serve every call whose table matches them (checked by
// checksum on the host side); a differing table -- a refit, a perturbed
// dataset -- is uploaded once into device memory with boys_table_create and
// evaluated by the run-time-order path below, whose operation sequence is
// the compiled path's (eval_point_uniform, bit-identical to the CPU oracle
// loaded with the same dataset).  Part of libboys.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstring>

#include "boys_device.cuh"
#include "boys_launch.h"

struct boys_table {
  boys_dtype dtype;
  int max_order;
  int device;
  void* rows_dev;
};

namespace boys {

// One point per thread.  nbar < 0: F_0..F_n from the order-n seed;
// otherwise eval_with_split (F_m, m > nbar, from the order-n seed and
// m <= nbar from the order-nbar seed).  AoS: the [256][n+1] tile is staged in
// shared memory and leaves as one bulk copy.
template <typename T, bool AOS>
__global__ void __launch_bounds__(kThreads)
table_kernel(const BoysRow<T>* __restrict__ rows, int n, int nbar, const T* __restrict__ X,
             int64_t N, T* __restrict__ out, T* __restrict__ expx, int64_t* __restrict__ dom,
             int64_t index_base, bool bulk_ok) {
  constexpr int NB = Tab<T>::MAX_ORDER;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* buf = reinterpret_cast<T*>(smem_raw);
  const int W = n + 1;
  const int tid = threadIdx.x;
  const PtrRows<T> R{rows};
  const int64_t ntiles = (N + kThreads - 1) / kThreads;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i0 = tile * kThreads;
    const int64_t i = i0 + tid;
    const bool in = i < N;
    const T x = in ? ldg_nc(X + i) : T(0);
    bool ok = valid_x(x);
    if (in && !ok) flag_domain(dom, index_base + i);
    ok = ok || !in;
    T* row = buf + tid * W;
    T* o = out + i;
    if (AOS) {
      if (tid == 0) bulk_wait_read<0>();
      __syncthreads();
    }
    auto put = [&](int m, T v) {
      if (AOS) row[m] = v;
      else if (in) __stcs(o + (int64_t)m * N, v);
    };
    const T t = eval_point_uniform<T, NB>(x, ok, n, R, [&](int m, T v) {
      if (m > nbar) put(m, v);
    });
    if (nbar >= 0) eval_point_uniform<T, NB>(x, ok, nbar, R, put);
    if (expx && in) __stcs(expx + i, t);
    if (AOS) {
      const int64_t cnt = (N - i0) < kThreads ? (N - i0) : kThreads;
      if (bulk_ok && cnt == kThreads) {
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) bulk_store(out + i0 * W, buf, (uint32_t)(kThreads * W * sizeof(T)));
      } else {
        __syncthreads();
        T* dst = out + i0 * W;
        for (int k = tid; k < cnt * W; k += kThreads) __stcs(dst + k, buf[k]);
      }
    }
  }
  if (AOS && tid == 0) bulk_wait_all();
}

template <typename T, bool AOS>
static boys_status launch_table(const void* rows, int n, int nbar, const void* x, int64_t N,
                                void* out, void* expx, int64_t* dom, int64_t base,
                                cudaStream_t s) {
  auto k = table_kernel<T, AOS>;
  const size_t smem = AOS ? (size_t)kThreads * (n + 1) * sizeof(T) : 0;
  static std::atomic<uint64_t> attr_mask{0};
  if (AOS) {
    boys_status st = opt_in_smem(
        k, (int)((size_t)kThreads * (Tab<T>::MAX_ORDER + 1) * sizeof(T)), attr_mask);
    if (st != BOYS_OK) return st;
  }
  const int64_t ntiles = (N + kThreads - 1) / kThreads;
  const bool bulk_ok = (reinterpret_cast<uintptr_t>(out) % 16) == 0;
  k<<<blocks_for(k, smem, ntiles), kThreads, smem, s>>>(
      (const BoysRow<T>*)rows, n, nbar, (const T*)x, N, (T*)out, (T*)expx, dom, base, bulk_ok);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_status(cudaGetLastError());
}

boys_status eval_table_base(const boys_table* tab, int n, int nbar, const void* x, int64_t N,
                            void* out, boys_layout lay, void* expx, int64_t* dom, int64_t base,
                            cudaStream_t s) {
  if (tab->dtype == BOYS_F64)
    return lay == BOYS_AOS ? launch_table<double, true>(tab->rows_dev, n, nbar, x, N, out, expx, dom, base, s)
                           : launch_table<double, false>(tab->rows_dev, n, nbar, x, N, out, expx, dom, base, s);
  return lay == BOYS_AOS ? launch_table<float, true>(tab->rows_dev, n, nbar, x, N, out, expx, dom, base, s)
                         : launch_table<float, false>(tab->rows_dev, n, nbar, x, N, out, expx, dom, base, s);
}

// Structural checks of an uploaded table: the run-time path's loops are
// bounded by the compiled tables' maximum factor counts and orders.
template <typename T>
static boys_status check_rows(const void* rows_host, int n_rows) {
  if (n_rows < 1 || n_rows > Tab<T>::MAX_ORDER + 1) return BOYS_E_ORDER;
  const BoysRow<T>* r = static_cast<const BoysRow<T>*>(rows_host);
  for (int k = 0; k < n_rows; ++k) {
    const int* c = r[k].cnt;
    if (c[0] < 0 || c[1] < 0 || c[2] < 0 || c[3] < 0) return BOYS_E_ARG;
    if (c[0] > MaxShape<T>::Q() || c[2] > MaxShape<T>::Q()) return BOYS_E_ARG;
    if (c[1] > MaxShape<T>::L() || c[3] > MaxShape<T>::L()) return BOYS_E_ARG;
  }
  return BOYS_OK;
}

}  // namespace boys

using namespace boys;

extern "C" {

size_t boys_table_row_bytes(boys_dtype dtype) {
  if (dtype == BOYS_F64) return sizeof(BoysRow<double>);
  if (dtype == BOYS_F32) return sizeof(BoysRow<float>);
  return 0;
}

const char* boys_table_checksum(boys_dtype dtype) {
  if (dtype == BOYS_F64) return BOYS_F64_TABLE_SHA256;
  if (dtype == BOYS_F32) return BOYS_F32_TABLE_SHA256;
  return "";
}

boys_status boys_table_create(boys_dtype dtype, const void* rows_host, int n_rows,
                              size_t row_bytes, boys_table** out) {
  if (!out || !rows_host) return BOYS_E_ARG;
  *out = nullptr;
  if (dtype != BOYS_F64 && dtype != BOYS_F32) return BOYS_E_DTYPE;
  if (row_bytes != boys_table_row_bytes(dtype)) return BOYS_E_ARG;
  boys_status st = dtype == BOYS_F64 ? check_rows<double>(rows_host, n_rows)
                                     : check_rows<float>(rows_host, n_rows);
  if (st != BOYS_OK) return st;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e);
  void* d = nullptr;
  e = cudaMalloc(&d, row_bytes * n_rows);
  if (e == cudaSuccess) e = cudaMemcpy(d, rows_host, row_bytes * n_rows, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(d);
    return cuda_status(e);
  }
  *out = new boys_table{dtype, n_rows - 1, dev, d};
  return BOYS_OK;
}

boys_status boys_table_destroy(boys_table* t) {
  if (!t) return BOYS_OK;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(t->device);
  cudaError_t e = cudaFree(t->rows_dev);
  cudaSetDevice(cur);
  delete t;
  return cuda_status(e);
}

int boys_table_max_order(const boys_table* t) { return t ? t->max_order : -1; }

boys_status boys_eval_dense_table(const boys_table* t, int n_max, const void* x_dev, int64_t N,
                                  void* out_dev, boys_layout layout, void* expx_dev,
                                  int64_t* dom_dev, void* stream) {
  if (!t) return BOYS_E_ARG;
  if (layout != BOYS_SOA && layout != BOYS_AOS) return BOYS_E_LAYOUT;
  if (n_max < 0 || n_max > t->max_order) return BOYS_E_ORDER;
  if (N < 0 || (N > 0 && (!x_dev || !out_dev))) return BOYS_E_ARG;
  if ((reinterpret_cast<uintptr_t>(x_dev) | reinterpret_cast<uintptr_t>(out_dev)) % dsize(t->dtype))
    return BOYS_E_ALIGN;
  if (N == 0) return BOYS_OK;
  return eval_table_base(t, n_max, -1, x_dev, N, out_dev, layout, expx_dev, dom_dev, 0,
                         (cudaStream_t)stream);
}

boys_status boys_eval_split_table(const boys_table* t, int n, int n_bar, const void* x_dev,
                                  int64_t N, void* out_dev, boys_layout layout, int64_t* dom_dev,
                                  void* stream) {
  if (!t) return BOYS_E_ARG;
  if (layout != BOYS_SOA && layout != BOYS_AOS) return BOYS_E_LAYOUT;
  if (n < 0 || n > t->max_order) return BOYS_E_ORDER;
  if (n_bar < 0 || n_bar >= n) return BOYS_E_ARG;
  if (N < 0 || (N > 0 && (!x_dev || !out_dev))) return BOYS_E_ARG;
  if ((reinterpret_cast<uintptr_t>(x_dev) | reinterpret_cast<uintptr_t>(out_dev)) % dsize(t->dtype))
    return BOYS_E_ALIGN;
  if (N == 0) return BOYS_OK;
  return eval_table_base(t, n, n_bar, x_dev, N, out_dev, layout, nullptr, dom_dev, 0,
                         (cudaStream_t)stream);
}

}  // extern "C"
