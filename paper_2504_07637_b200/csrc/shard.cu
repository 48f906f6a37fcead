// Per-shard error statistic (component `shard_error_reduce`):
// the max relative error of this shard's own outputs at the positions where
// reference values were spliced into its inputs, reduced on the device into
// one fp64 that the multi-GPU driver all-gathers (8 bytes per rank).  Part of
// libboys.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "boys_device.cuh"
#include "boys_launch.h"

namespace boys {

// rel_j = |(v - hi) - lo| / max(|hi|, tiny): relative error, measured
// against the dtype's smallest normal where the true value is below it
// (tests/accuracy.py rel_err); NaN -> +inf.  Max over j, folded into *err
// with an integer atomicMax on the bit pattern (monotonic for values >= 0).
template <typename T>
__global__ void __launch_bounds__(kThreads)
shard_error_kernel(const T* __restrict__ vals, const int64_t* __restrict__ pos,
                   const double* __restrict__ gold, int64_t K, double tiny,
                   double* __restrict__ err) {
  __shared__ double s[kThreads / 32];
  double m = 0.0;
  for (int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x; j < K;
       j += (int64_t)gridDim.x * kThreads) {
    const double v = (double)vals[pos[j]];
    const double hi = gold[2 * j], lo = gold[2 * j + 1];
    const double e = fabs((v - hi) - lo);
    double r = e / fmax(fabs(hi), tiny);
    if (isnan(r)) r = __longlong_as_double(0x7ff0000000000000LL);
    m = fmax(m, r);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) m = fmax(m, __shfl_xor_sync(kFull, m, d));
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kThreads / 32; ++w) m = fmax(m, s[w]);
    atomicMax(reinterpret_cast<unsigned long long*>(err),
              (unsigned long long)__double_as_longlong(m));
  }
}

boys_status shard_error_base(boys_dtype dtype, const void* vals, const int64_t* pos,
                             const double* gold, int64_t K, double* err, cudaStream_t s) {
  if (K == 0) return BOYS_OK;
  const int64_t blocks64 = (K + kThreads - 1) / kThreads;
  const int blocks = (int)(blocks64 < 2 * sm_count() ? blocks64 : 2 * sm_count());
  if (dtype == BOYS_F64)
    shard_error_kernel<double><<<blocks, kThreads, 0, s>>>((const double*)vals, pos, gold, K,
                                                           0x1p-1022, err);
  else
    shard_error_kernel<float><<<blocks, kThreads, 0, s>>>((const float*)vals, pos, gold, K,
                                                          0x1p-126, err);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_status(cudaGetLastError());
}

}  // namespace boys
