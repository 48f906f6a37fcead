// Host-side launch plumbing shared by the libboys translation units: error
// state, SM count, shared-memory opt-in, cached occupancy, the A/B knobs, and
// the per-family entry points each .cu file exports to the C ABI (abi.cu).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "../../include/boys.h"

namespace boys {

constexpr int kLaunchThreads = 256;          // == kThreads (boys_device.cuh)
extern std::atomic<int64_t> g_launches;      // kernels launched (boys_launch_count)
extern thread_local char g_cuda_err[256];    // last CUDA error text (per host thread)

inline size_t dsize(boys_dtype d) { return d == BOYS_F64 ? 8 : 4; }

// ---------------------------------------------------------------------------
// launch plumbing
// ---------------------------------------------------------------------------
inline int sm_count() {
  int dev = 0, v = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  return v;
}

inline boys_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return BOYS_OK;
  snprintf(g_cuda_err, sizeof g_cuda_err, "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
  return BOYS_E_CUDA;
}

// Persistent grid: SMs x resident blocks (measured better than one block per
// tile even for the 2^20-point config: block launch overhead dominates there).
// Opt a kernel in to more than 48 KB of dynamic shared memory on the current
// device (the attribute is per device; `mask` remembers which devices are done).
template <typename K>
inline boys_status opt_in_smem(K kernel, int smem, std::atomic<uint64_t>& mask) {
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

// The occupancy query is cached per (device, kernel, shared memory, block
// size): it is a host-side call that would otherwise sit on every launch's
// critical path.  64 slots per host thread cover every kernel of the library
// in use at once; past that the query simply runs again.
template <typename K>
inline int blocks_for(K kernel, size_t smem, int64_t ntiles, int threads = kLaunchThreads) {
  struct Slot { const void* k; size_t smem; int threads, dev, occ, sms; };
  static thread_local Slot cache[64] = {};
  static thread_local int next = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const void* key = reinterpret_cast<const void*>(kernel);
  const Slot* hit = nullptr;
  for (const Slot& c : cache)
    if (c.k == key && c.smem == smem && c.threads == threads && c.dev == dev) { hit = &c; break; }
  if (!hit) {
    int occ = 0, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cache[next] = Slot{key, smem, threads, dev, occ < 1 ? 1 : occ, sms};
    hit = &cache[next];
    next = (next + 1) % 64;
  }
  int64_t b = (int64_t)hit->sms * hit->occ;
  if (ntiles < b) b = ntiles;
  return (int)(b < 1 ? 1 : b);
}

// Ragged grid = resident blocks x this: f64 persistent (x1: 1.90 ms; x2 1.90,
// x4 1.91, x16 1.98), f32 x4 (0.984 vs 1.007 ms at x1), same-box cfg4 sweep.
inline int ragged_grid_mult(bool f64) { return f64 ? 1 : 4; }
// Host-buffer pipelines: elements per chunk (2^22: the PCIe link bounds the
// pipeline; larger chunks measured no faster).
constexpr int64_t kHostChunk = int64_t(1) << 22;

// per-family entry points (dense.cu, split.cu, ragged.cu)
boys_status eval_dense_base(boys_dtype dtype, int n_max, const void* x, int64_t N, void* out,
                            boys_layout lay, void* expx, int64_t* dom, int64_t base,
                            cudaStream_t s);
boys_status eval_split_base(boys_dtype dtype, int n, int n_bar, const void* x, int64_t N,
                            void* out, boys_layout lay, int64_t* dom, cudaStream_t s);
boys_status eval_ragged_base(boys_dtype dtype, const void* x, const uint8_t* nm,
                             const int64_t* off, int64_t N, void* out, int64_t* dom,
                             cudaStream_t s);
boys_status ragged_offsets_base(const uint8_t* nm, int64_t N, int64_t* off, cudaStream_t s);
boys_status hermite_base(int L, const double* bra, int64_t Nb, const double* ket, int64_t Nk,
                         double* out, int64_t* dom, cudaStream_t s);
boys_status shard_error_base(boys_dtype dtype, const void* vals, const int64_t* pos,
                             const double* gold, int64_t K, double* err, cudaStream_t s);

}  // namespace boys
