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
  static int sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return sms;
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

// The occupancy query is cached per (kernel, shared-memory size): it is a
// host-side call that would otherwise sit on every launch's critical path.
template <typename K>
inline int blocks_for(K kernel, size_t smem, int64_t ntiles, int threads = kLaunchThreads) {
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
inline int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}
inline int aos_nbuf() {
  static int v = env_int("BOYS_AOS_NBUF", 2) == 1 ? 1 : 2;
  return v;
}
inline int soa_tma() {   // BOYS_SOA_TMA=1: SoA rows leave as bulk copies
  static int v = env_int("BOYS_SOA_TMA", 0);
  return v;
}
inline int grid_tiles() {
  static int v = env_int("BOYS_GRID_TILES", 0);
  return v;
}
inline int soa_small_minb() {   // BOYS_SOA0_MINB: 8 (default) or 6 for n <= 1
  static int v = env_int("BOYS_SOA0_MINB", 8) == 6 ? 6 : 8;
  return v;
}
inline int soa_pair() {   // BOYS_SOA_PAIR=1: two adjacent points per thread (SoA)
  static int v = env_int("BOYS_SOA_PAIR", 1);
  return v;
}
// Grid for the paired SoA kernel (BOYS_PAIR_GRID: 0 = rule below, 1 = per
// tile, 2 = persistent).  Same-box sweeps (tools/ab/ab33.sh, 2^24 points):
// one block per 512-point tile wins for every f64 order (n=8: 230 vs 266 us,
// n=12: 314 vs 371 us) and for f32 n >= 6 (n=8: 112 vs 132 us); persistent
// for f32 n < 6 (n=4: 82 vs 90 us).
inline bool soa_pair_per_tile(bool f64, int n) {
  static int v = env_int("BOYS_PAIR_GRID", 0);
  if (v) return v == 1;
  return f64 || n >= 6;
}
// Ragged grid = resident blocks x this (BOYS_RAGGED_GRID_MULT overrides).
// Same-box sweep (tools/ab/ab35.sh, cfg4): f64 best persistent (x1: 1.90 ms;
// x2 1.90, x4 1.91, x16 1.98); f32 best x4 (0.984 vs 1.007 ms at x1).
inline int ragged_grid_mult(bool f64) {
  static int v = env_int("BOYS_RAGGED_GRID_MULT", 0);
  if (v >= 1) return v;
  return f64 ? 1 : 4;
}
// AoS with two points per thread (dense_aos_pair_kernel): by default where the
// double-buffered 512-point tile allows 3 blocks/SM (f64 n <= 8, every f32
// order): f64 n=2: 168 vs 196 us, n=8: 241 vs 248 us; f32 n=8: 116 vs 144 us,
// n=16: 197 vs 217 us at 2^24 (tools/ab/ab47.sh, ab48.sh); slower for f64
// n >= 10 (cfg5 n=12: 1.30 vs 1.25 ms).  BOYS_AOS_PAIR=0/1 forces it off/on.
inline bool aos_pair(bool small_tile) {
  static int v = env_int("BOYS_AOS_PAIR", -1);
  return v < 0 ? small_tile : v == 1;
}
// SoA with four adjacent points per thread (dense_soa_quad_kernel): default for
// n <= 3 (f64 2^24: n=0 113 vs 123 us, n=1 122 vs 135, n=3 152 vs 167; f32
// n <= 2 9-13% faster; n=4 neutral, n=5 slower; tools/ab/ab49.sh, ab50.sh).
// BOYS_SOA_QUAD=0/1 forces it off/on (on: orders up to 5).
inline bool soa_quad(int n) {
  static int v = env_int("BOYS_SOA_QUAD", -1);
  return v < 0 ? n <= 3 : v == 1;
}
// Host-buffer pipelines: elements per chunk (BOYS_HOST_CHUNK_LOG2, default 22).
inline int64_t host_chunk() {
  static int64_t v = int64_t(1) << env_int("BOYS_HOST_CHUNK_LOG2", 22);
  return v;
}
// Register-row AoS kernel for n = 1, 3 (dense_aos_vec_kernel); BOYS_AOS_VEC=0/1
// forces it off/on, otherwise the per-(dtype, order) default from dense.cu.
inline bool aos_vec(bool deflt) {
  static int v = env_int("BOYS_AOS_VEC", -1);
  return v < 0 ? deflt : v == 1;
}
inline int pdl() {   // BOYS_PDL=0: plain stream-serialised launches (A/B)
  static int v = env_int("BOYS_PDL", 1);
  return v;
}
inline int aos_minb() {
  static int v = env_int("BOYS_AOS_MINB", 4) == 6 ? 6 : 4;
  return v;
}

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
boys_status shard_error_base(boys_dtype dtype, const void* vals, const int64_t* pos,
                             const double* gold, int64_t K, double* err, cudaStream_t s);

}  // namespace boys
