// Microbenchmark: dependent-chain latency and issue behaviour of DFMA/DMUL/SEL on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP, int MODE>
__global__ void chain(double* out, const double* in, int iters, long long* cyc) {
  double a[ILP], b = in[1], c = in[2];
  int n = (int)in[3];
#pragma unroll
  for (int k = 0; k < ILP; ++k) a[k] = in[0] + k + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int k = 0; k < ILP; ++k) {
        if (MODE == 0) a[k] = __fma_rn(a[k], b, c);
        if (MODE == 1) a[k] = __dmul_rn(__fma_rn(a[k], b, c), b);
        if (MODE == 2) { double nx = __dmul_rn(__fma_rn(a[k], b, c), b); a[k] = (i * 8 + u < n + k) ? nx : a[k]; }
      }
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int ILP, int MODE>
void run(int warps, const char* name) {
  double *out, *in; long long* cyc;
  cudaMalloc(&out, 1 << 20); cudaMalloc(&in, 64); cudaMalloc(&cyc, 8);
  double h[4] = {1.0, 0.999999, 1e-9, 1e9};
  cudaMemcpy(in, h, 32, cudaMemcpyHostToDevice);
  const int iters = 2000;
  chain<ILP, MODE><<<1, 32 * warps>>>(out, in, iters, cyc);
  chain<ILP, MODE><<<1, 32 * warps>>>(out, in, iters, cyc);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const int per = MODE == 0 ? 1 : MODE == 1 ? 2 : 2;
  printf("%s ilp=%d warps=%d: %.2f cycles per chain step (%d DP ops), %.2f cyc per DP warp-instr per SMSP\n", name, ILP, warps,
         (double)c / (iters * 8), per, (double)c / (iters * 8) / (per * ILP) / ((warps + 3) / 4));
  cudaFree(out); cudaFree(in); cudaFree(cyc);
}
int main() {
  run<1, 0>(1, "dfma"); run<2, 0>(1, "dfma"); run<4, 0>(1, "dfma"); run<8, 0>(1, "dfma");
  run<1, 0>(4, "dfma"); run<4, 0>(4, "dfma"); run<4, 0>(16, "dfma"); run<4,0>(32,"dfma");
  run<1, 1>(1, "dfma+dmul"); run<3, 1>(1, "dfma+dmul"); run<3, 1>(16, "dfma+dmul");
  run<1, 2>(1, "dfma+dmul+sel"); run<3, 2>(1, "dfma+dmul+sel"); run<3, 2>(16, "dfma+dmul+sel"); run<3, 2>(32, "dfma+dmul+sel");
  return 0;
}
