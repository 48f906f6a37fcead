// Fused consumer (SPEC.md:16, 353 name downstream integral
// code as the Boys functions' caller): McMurchie-Davidson Hermite Coulomb
// integrals for a batch of primitive bra pairs x ket pairs.  Each thread owns
// one quartet (bra pair i, ket pair j):
//   a = p q / (p + q),  x = a |P - Q|^2,
//   F_0..F_L(x)                       the Boys evaluator, kept in registers
//   R^{(n)}_{000} = (-2a)^n F_n(x)
//   R^{(n)}_{t+1,u,v} = t R^{(n+1)}_{t-1,u,v} + X_PQ R^{(n+1)}_{t,u,v}   (and u, v)
//   out = pref R^{(0)}_{tuv},  pref = 2 pi^{5/2} / (p q sqrt(p + q)) K_i K_j
// for the (L+1)(L+2)(L+3)/6 Hermite indices t+u+v <= L.  F_m never reaches
// HBM.  The recursion runs in place over one register array, level n = L-1
// .. 0, each level in decreasing total order s = t+u+v (a level-n entry of
// order s reads level-(n+1) entries of order s-1 and s-2, not yet
// overwritten).  Operation order is fixed (explicit fma/mul/div/sqrt) and
// restated by the CPU oracle in oracle/ (its Hermite entry):
// bit-identical.  Part of libboys.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "boys_device.cuh"
#include "boys_launch.h"

namespace boys {

// canonical Hermite index: s = t+u+v ascending; within s, t descending, then
// u descending (v = s - t - u)
__host__ __device__ constexpr int herm_count(int L) { return (L + 1) * (L + 2) * (L + 3) / 6; }
__host__ __device__ constexpr int herm_index(int t, int u, int v) {
  const int s = t + u + v;
  int before = 0;
  for (int tp = s; tp > t; --tp) before += s - tp + 1;
  return herm_count(s - 1) + before + (s - t - u);
}

constexpr double kTwoPi52 = 0x1.17e50a9dc6553p+5;   // RN(2 pi^{5/2}) = 34.986836655249725

template <int L>
__device__ __forceinline__ void hermite_quartet(const double* __restrict__ bra,
                                                const double* __restrict__ ket, bool ok_in,
                                                double (&R)[herm_count(L)], bool& ok) {
  using A = Ar<double>;
  const double p = bra[0], q = ket[0];
  const double X = A::sub(bra[1], ket[1]), Y = A::sub(bra[2], ket[2]), Z = A::sub(bra[3], ket[3]);
  const double pq = A::add(p, q);
  const double a = A::div(A::mul(p, q), pq);
  const double r2 = A::fma(Z, Z, A::fma(Y, Y, A::mul(X, X)));
  const double x = A::mul(a, r2);
  ok = ok_in && valid_x(x) && p > 0.0 && q > 0.0;
  double F[L + 1];
  eval_point_stream<double, L>(x, ok, [&](int m, double v) { F[m] = v; });
  const double m2a = A::mul(-2.0, a);
  double R0[L + 1];
  double pw = 1.0;
#pragma unroll
  for (int k = 0; k <= L; ++k) {
    R0[k] = A::mul(pw, F[k]);
    pw = A::mul(pw, m2a);
  }
  R[0] = R0[L];
#pragma unroll
  for (int n = L - 1; n >= 0; --n) {
#pragma unroll
    for (int s = L - n; s >= 1; --s) {
#pragma unroll
      for (int t = s; t >= 0; --t) {
#pragma unroll
        for (int u = s - t; u >= 0; --u) {
          const int v = s - t - u;
          double val;
          if (t > 0) {
            val = t >= 2 ? A::fma(X, R[herm_index(t - 1, u, v)],
                                  A::mul(double(t - 1), R[herm_index(t >= 2 ? t - 2 : 0, u, v)]))
                         : A::mul(X, R[herm_index(t - 1, u, v)]);
          } else if (u > 0) {
            val = u >= 2 ? A::fma(Y, R[herm_index(0, u - 1, v)],
                                  A::mul(double(u - 1), R[herm_index(0, u >= 2 ? u - 2 : 0, v)]))
                         : A::mul(Y, R[herm_index(0, u - 1, v)]);
          } else {
            val = v >= 2 ? A::fma(Z, R[herm_index(0, 0, v - 1)],
                                  A::mul(double(v - 1), R[herm_index(0, 0, v >= 2 ? v - 2 : 0)]))
                         : A::mul(Z, R[herm_index(0, 0, v - 1)]);
          }
          R[herm_index(t, u, v)] = val;
        }
      }
    }
    R[0] = R0[n];
  }
  const double den = A::mul(A::mul(p, q), A::sqrt(pq));
  const double pref = A::mul(A::mul(A::div(kTwoPi52, den), bra[4]), ket[4]);
#pragma unroll
  for (int k = 0; k < herm_count(L); ++k) R[k] = A::mul(pref, R[k]);
}

// Persistent grid over tiles of 128 quartets (flat index q = i Nk + j); each
// tile's [128][NH] outputs are staged in shared memory (odd NH: conflict-free
// 64-bit banks; even NH: 2-way) and leave as one bulk async copy, double-
// buffered.  Pair records are 5 doubles (p, Px, Py, Pz, K).
template <int L>
__global__ void __launch_bounds__(128)
hermite_kernel(const double* __restrict__ bra, int64_t Nb, const double* __restrict__ ket,
               int64_t Nk, double* __restrict__ out, int64_t* __restrict__ dom, bool bulk_ok) {
  constexpr int NH = herm_count(L), TILE = 128, TILE_ELEMS = TILE * NH;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sbase = reinterpret_cast<double*>(smem_raw);
  const int tid = threadIdx.x;
  const int64_t NQ = Nb * Nk;
  const int64_t ntiles = (NQ + TILE - 1) / TILE;
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int64_t q0 = tile * TILE, qi = q0 + tid;
    const bool in = qi < NQ;
    const int64_t i = in ? qi / Nk : 0, j = in ? qi - i * Nk : 0;
    double R[NH];
    bool ok;
    hermite_quartet<L>(bra + 5 * i, ket + 5 * j, true, R, ok);
    if (in && !ok) flag_domain(dom, qi);
    double* buf = sbase + (it & 1) * TILE_ELEMS;
    if (tid == 0) bulk_wait_read<1>();
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NH; ++k) buf[tid * NH + k] = R[k];
    const int64_t cnt = (NQ - q0) < TILE ? (NQ - q0) : TILE;
    if (bulk_ok && cnt == TILE) {
      fence_proxy_async_smem();
      __syncthreads();
      if (tid == 0) bulk_store(out + q0 * NH, buf, TILE_ELEMS * sizeof(double));
    } else {
      __syncthreads();
      double* dst = out + q0 * NH;
      for (int k = tid; k < cnt * NH; k += TILE) __stcs(dst + k, buf[k]);
    }
  }
  if (tid == 0) bulk_wait_all();
}

template <int L>
static boys_status launch_hermite(const double* bra, int64_t Nb, const double* ket, int64_t Nk,
                                  double* out, int64_t* dom, cudaStream_t s) {
  auto k = hermite_kernel<L>;
  const size_t smem = 2 * 128 * herm_count(L) * sizeof(double);
  static std::atomic<uint64_t> attr_mask{0};
  boys_status st = opt_in_smem(k, (int)smem, attr_mask);
  if (st != BOYS_OK) return st;
  const int64_t ntiles = (Nb * Nk + 127) / 128;
  const bool bulk_ok = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  k<<<blocks_for(k, smem, ntiles, 128), 128, smem, s>>>(bra, Nb, ket, Nk, out, dom, bulk_ok);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_status(cudaGetLastError());
}

boys_status hermite_base(int L, const double* bra, int64_t Nb, const double* ket, int64_t Nk,
                         double* out, int64_t* dom, cudaStream_t s) {
  switch (L) {
    case 0: return launch_hermite<0>(bra, Nb, ket, Nk, out, dom, s);
    case 1: return launch_hermite<1>(bra, Nb, ket, Nk, out, dom, s);
    case 2: return launch_hermite<2>(bra, Nb, ket, Nk, out, dom, s);
    case 3: return launch_hermite<3>(bra, Nb, ket, Nk, out, dom, s);
    case 4: return launch_hermite<4>(bra, Nb, ket, Nk, out, dom, s);
    default: return BOYS_E_ORDER;
  }
}

}  // namespace boys
