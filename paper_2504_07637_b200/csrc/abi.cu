// libboys (include/boys.h): the C ABI and the host-buffer pipelines.  Kernels:
// dense.cu, ragged.cu, split.cu; shared device code: boys_device.cuh.
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
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/boys.h"
#include "boys_launch.h"
#include "boys_eval.cuh"   // table bounds (BOYS_F64_MAX_ORDER / BOYS_F32_MAX_ORDER)

#ifndef BOYS_VERSION
#define BOYS_VERSION "0.2.0"
#endif

namespace boys {

std::atomic<int64_t> g_launches{0};
thread_local char g_cuda_err[256] = "";

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
  return eval_split_base(dtype, n, n_bar, x_dev, N, out_dev, layout, dom_dev,
                         (cudaStream_t)stream);
}

boys_status boys_eval_ragged(boys_dtype dtype, const void* x_dev, const uint8_t* nmax_dev,
                             const int64_t* offsets_dev, int64_t N, void* out_dev,
                             int64_t* dom_dev, void* stream) {
  if (dtype != BOYS_F64 && dtype != BOYS_F32) return BOYS_E_DTYPE;
  if (N < 0) return BOYS_E_ARG;
  if (N == 0) return BOYS_OK;
  if (!x_dev || !nmax_dev || !offsets_dev || !out_dev) return BOYS_E_ARG;
  // element alignment (the kernel derives the 16-byte phase from the address)
  if ((reinterpret_cast<uintptr_t>(x_dev) | reinterpret_cast<uintptr_t>(out_dev)) % dsize(dtype) ||
      reinterpret_cast<uintptr_t>(offsets_dev) % sizeof(int64_t))
    return BOYS_E_ALIGN;
  return eval_ragged_base(dtype, x_dev, nmax_dev, offsets_dev, N, out_dev, dom_dev,
                          (cudaStream_t)stream);
}

boys_status boys_ragged_offsets(const uint8_t* nmax_dev, int64_t N, int64_t* offsets_dev,
                                void* stream) {
  if (N < 0 || !offsets_dev || (N > 0 && !nmax_dev)) return BOYS_E_ARG;
  return ragged_offsets_base(nmax_dev, N, offsets_dev, (cudaStream_t)stream);
}

boys_status boys_shard_error(boys_dtype dtype, const void* vals_dev, const int64_t* pos_dev,
                             const double* gold_dev, int64_t K, double* err_dev, void* stream) {
  if (dtype != BOYS_F64 && dtype != BOYS_F32) return BOYS_E_DTYPE;
  if (K < 0 || !err_dev || (K > 0 && (!vals_dev || !pos_dev || !gold_dev))) return BOYS_E_ARG;
  return shard_error_base(dtype, vals_dev, pos_dev, gold_dev, K, err_dev, (cudaStream_t)stream);
}

boys_status boys_hermite_coulomb(int L, const double* bra_dev, int64_t Nb, const double* ket_dev,
                                 int64_t Nk, double* out_dev, int64_t* dom_dev, void* stream) {
  if (L < 0 || L > 4) return BOYS_E_ORDER;
  if (Nb < 0 || Nk < 0) return BOYS_E_ARG;
  if (Nb == 0 || Nk == 0) return BOYS_OK;
  if (!bra_dev || !ket_dev || !out_dev) return BOYS_E_ARG;
  if ((reinterpret_cast<uintptr_t>(bra_dev) | reinterpret_cast<uintptr_t>(ket_dev) |
       reinterpret_cast<uintptr_t>(out_dev)) % sizeof(double))
    return BOYS_E_ALIGN;
  if (Nb > (int64_t(1) << 62) / Nk) return BOYS_E_ARG;
  return hermite_base(L, bra_dev, Nb, ket_dev, Nk, out_dev, dom_dev, (cudaStream_t)stream);
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
  const int64_t chunk = N < kHostChunk ? N : kHostChunk;
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
  const int64_t chunk = N < kHostChunk ? N : kHostChunk;
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
    st = eval_ragged_base(dtype, p->dx[k], p->dn[k], p->doff[k], cn, p->dout[k], p->ddom + c, s);
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
