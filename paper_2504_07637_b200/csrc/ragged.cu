// Ragged batches (per-element order) and their offsets scan.  Part of libboys.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <type_traits>

#include "boys_device.cuh"
#include "boys_launch.h"

namespace boys {

// ---------------------------------------------------------------------------
// ragged kernel: element i, order n_i, values at out[offsets[i] + m]
//
// Warp-autonomous (no block barriers): each warp walks full chunks of 32*EPL
// elements (the batch's last partial chunk goes per element at the end).
//   * every lane: e^{-x}; elements past their cut-off (x >= z_{n_i}, ~95% of
//     ERI-like batches) run the cheap run-time-order tail at once into the
//     warp's staging slot -- seed, then the recursion entered once through a
//     jump table on the warp's maximum order -- and the chunk's contiguous
//     output range leaves as one bulk copy (plus scalar head/tail elements).
//   * elements below their cut-off are deferred to a warp-private queue and
//     evaluated 32 at a time with every lane busy (Q~ is the expensive part),
//     each lane writing its element's n+1 values directly (ragged_drain).
// Values are bit-identical to boys_eval_dense at each element's order.
// The kernel is instruction-issue bound (ncu: DRAM bytes = algorithmic bytes);
// what the round-2 profiles changed is listed in DESIGN.md section 5.
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
  // deferred elements: x and (order << 56 | offset); the drain recomputes
  // e^{-x}.  Two stores per element slot in the chunk pass (x, t, order and
  // offset separately: four; the element index alone: one, but the drain's
  // dependent reloads then showed up as long-scoreboard stalls).
  T qx[QCAP];
  int64_t qon[QCAP];
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

// (Two queued elements per lane, 64 per call, so that a lane's two chains
// interleave: 1.54 vs 1.42 ms f64, 0.79 vs 0.75 ms f32.)
// Evaluate up to 32 queued elements (one per lane), writing straight to
// global memory; returns the new queue length.  Out of line: it runs once per
// ~7 chunks of an ERI-like batch, and inlined into the chunk loop its
// constants (22 uniform loads) and registers were paid on every chunk.
template <typename T, int NB, typename WarpT>
__device__ __noinline__ int ragged_drain(WarpT& W, SmemRows<T> st, int qn, T* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  // queued elements' slots were written (with stale staging data) by earlier
  // bulk stores of their chunks: those must be complete before we overwrite
  if (lane == 0) bulk_wait_all();
  __syncwarp();
  const int take = qn < 32 ? qn : 32;
  const bool has = lane < take;
  const int slot = qn - take + lane;            // LIFO: the newest `take` entries
  const T x = has ? W.qx[slot] : T(0);
  const int64_t on = has ? W.qon[slot] : 0;
  const int n = (int)(on >> 56);
  const int64_t off = on & ((int64_t(1) << 56) - 1);
  const T t = exp_neg_select(x);
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
  return qn - take;
}

// high word of the bit pattern (fp64) / the bit pattern (fp32)
__device__ __forceinline__ unsigned hi_word(double v) { return (unsigned)__double2hiint(v); }
__device__ __forceinline__ unsigned hi_word(float v) { return __float_as_uint(v); }

// Chunk-path test on x, one integer compare: fp64 -- positive, finite and
// below `bound_hi` (the high word of the smallest staged x_up, a power of
// two), so the upward ladder is not needed; fp32 -- positive and finite
// (x > x_up joins the queue there).  -0.0 fails it and takes the general path.
template <typename T>
__device__ __forceinline__ bool hot_x(T x, unsigned bound_hi) {
  return hi_word(x) < (sizeof(T) == 8 ? bound_hi : 0x7f800000u);
}

// General per-element path (kept out of line: it is cold and large): element
// `idx` evaluated from the __constant__ rows at any tabulated order and
// written directly at its offset; NaN row and domain flag for invalid x or an
// order above the table.
template <typename T>
__device__ __noinline__ void ragged_general_element(T x, int n, int64_t goff, bool in, int64_t idx,
                                                    T* __restrict__ out, int64_t* __restrict__ dom) {
  constexpr int MAXN = Tab<T>::MAX_ORDER;
  const bool okl = in && valid_x(x) && n <= MAXN;
  if (in && !okl) {
    flag_domain(dom, idx);
    for (int m = 0; m <= n; ++m) out[goff + m] = Ar<T>::nan();
  }
  T* dst = out + goff;
  eval_point_rt<T, MAXN>(x, okl, okl ? n : 0, ConstRows<T>{}, [&](int m, T v) {
    if (okl) dst[m] = v;
  });
}

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
  const int64_t nfull = N / CH;                  // full chunks: the loop below
  const int64_t wstride = (int64_t)gridDim.x * (WT / 32);
  int qn = 0;                                    // warp-uniform queue length
  int64_t c = (int64_t)blockIdx.x * (WT / 32) + wid;
  // software pipeline: inputs of the warp's next chunk are loaded one
  // iteration ahead through running pointers (lane's first element of it)
  const T* xp = X + c * CH + lane;
  const uint8_t* np = NM + c * CH + lane;
  const int64_t* op = OFF + c * CH + lane;
  const int64_t pstep = wstride * CH;
  // Prefetch of the warp's next chunk, two ways (same-box A/B, cfg4):
  //  * fp64 (kTwoSets): a second register set loaded at the top of the
  //    iteration, a whole iteration ahead, and copied at the next top.  With 16
  //    warps per SM the shorter distance below left long-scoreboard stalls at
  //    the loop top (1.53-1.60 vs 1.50 ms) although it issues 8% fewer
  //    instructions.
  //  * fp32: x / n / goff themselves are reloaded in the middle of the
  //    iteration, right after their last use (before the recursion steps): no
  //    second set, no copies, 70 registers, so three blocks per SM hide the
  //    shorter distance (0.775 vs 0.873 ms; loading earlier, after the enqueue,
  //    needs 83 registers: 0.81-0.86 ms).
  constexpr bool kTwoSets = sizeof(T) == 8;
  T x[EPL], px[EPL];
  int n[EPL], pn[EPL];
  int64_t goff[EPL], poff[EPL], last_off = 0, plast_off = 0;
  auto load = [&](T (&lx)[EPL], int (&ln)[EPL], int64_t (&lo)[EPL], int64_t& llast) {
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      lx[e] = ldg_nc(xp + 32 * e);
      ln[e] = (int)np[32 * e];
      lo[e] = __ldg(op + 32 * e);
    }
    llast = __ldg(op + (CH - lane));             // OFF[first + CH]: the range's end
  };
  // next chunk of this warp: advance, and load its inputs if it is a full one
  bool have;
  auto advance = [&]() {
    c += wstride;
    xp += pstep;
    np += pstep;
    op += pstep;
    have = c < nfull;
    if (have) {
      if (kTwoSets) load(px, pn, poff, plast_off);
      else load(x, n, goff, last_off);
    }
    // fp32: L2 prefetch of the chunk after that one (one 32-byte sector per lane
    // and array where the chunk has that many): the mid-iteration reload then
    // hits L2 (0.751 -> 0.742 ms; fp64: with either prefetch form 1.44-1.47 vs
    // 1.42 ms)
    if (!kTwoSets && c + wstride < nfull) {
      constexpr int XS = CH * (int)sizeof(T) / 32, OS = CH * 8 / 32, NS = (CH + 31) / 32;
      const int64_t j1 = (c + wstride) * CH;
      if (lane < OS) prefetch_l2(OFF + j1 + lane * 4);
      if (lane < XS) prefetch_l2(X + j1 + lane * (32 / (int)sizeof(T)));
      if (lane < NS) prefetch_l2(NM + j1 + lane * 32);
    }
  };
  // hot-path bound on x: below every staged order's x_up (fp64: the upward
  // ladder then never runs in the chunk path; such x take the general path)
  unsigned xup_hi_min = 0x7ff00000u;
  if (!kDeferUp<T>) {
    for (int k = 0; k <= NB; ++k) xup_hi_min = min(xup_hi_min, hi_word(Tab<T>::row(k).x_up));
  }
  const unsigned lt_mask = (1u << lane) - 1u;
  have = c < nfull;
  if (have) {
    if (kTwoSets) load(px, pn, poff, plast_off);
    else load(x, n, goff, last_off);
  }
  while (have) {
    const int64_t il = c * CH + lane;            // the lane's first element
    if (kTwoSets) {
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        x[e] = px[e];
        n[e] = pn[e];
        goff[e] = poff[e];
      }
      last_off = plast_off;
      advance();
    }
    // the range's start OFF[c * CH] is lane 0's first offset
    const int64_t base = __shfl_sync(kFull, goff[0], 0), cnt = last_off - base;
    // The chunk path below assumes a full chunk of valid elements (x finite,
    // >= 0 and, in fp64, below x_up; order <= NB) whose offsets are the prefix
    // sum of n + 1 and whose output range fits the staging slot.  Anything else
    // -- invalid x or orders, gapped offsets,
    // orders above the fast path's bound -- takes the general per-element path.
    bool slow = cnt > WarpT::CAP;
    int cnt_l = 0;
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      slow = slow || !hot_x<T>(x[e], xup_hi_min) || n[e] > NB;
      cnt_l += n[e] + 1;
    }
    const int64_t cnt_sum = (int64_t)__reduce_add_sync(kFull, (unsigned)cnt_l);   // every lane
    slow = slow || cnt_sum != cnt;
    if (__any_sync(kFull, slow)) {
#pragma unroll
      for (int e = 0; e < EPL; ++e)
        ragged_general_element<T>(x[e], n[e], goff[e], true, il + 32 * e, out, dom);
      if (!kTwoSets) advance();
      continue;
    }
    // staging position matches the global 16-byte phase of the chunk range
    constexpr int Q = 16 / sizeof(T);
    // (from the address: `out` need only be element-aligned)
    const int shift = (int)((reinterpret_cast<uintptr_t>(out + base) / sizeof(T)) & (Q - 1));
    // the previous chunk's bulk store must have finished reading the slot
    if (lane == 0) bulk_wait_read<0>();
    __syncwarp();
    T t[EPL], cur[EPL], tx[EPL];
    ZcRow<T> zc[EPL];
    T* dst[EPL];
    bool wr[EPL];
    int wmax_l = 0;
    // The math below is written phase by phase over all EPL elements with no
    // branch between the elements of a phase, so each phase is one basic block
    // and the elements' independent dependency chains interleave (FP64: 8-cycle
    // DFMA latency; element-by-element code left the warp waiting on one chain).
    // (evaluating e^{-x} only for the elements with x <= XEXP, compacted one
    // per lane, measured no faster: tools/ab/ab24.sh)
#pragma unroll
    for (int e = 0; e < EPL; ++e) zc[e] = S.zc[n[e]];
#pragma unroll
    for (int e = 0; e < EPL; ++e) t[e] = exp_neg_select(x[e]);
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      // deferred to the warp queue: below the cut-off (Q~ needed) and, in
      // fp32, above x_up (upward ladder).  Branch-free enqueue; qn stays
      // warp-uniform.
      const bool defer = x[e] < zc[e].z || (kDeferUp<T> && x[e] > zc[e].x_up);
      const unsigned dmask = __ballot_sync(kFull, defer);
      dst[e] = W.stage + (int)(goff[e] - base) + shift;
      const int slot = qn + __popc(dmask & lt_mask);
      psts(defer, &W.qx[slot], x[e]);
      psts(defer, &W.qon[slot], goff[e] | ((int64_t)n[e] << 56));   // one op on the high word
      qn += __popc(dmask);
      wr[e] = !defer;
      wmax_l = max(wmax_l, defer ? 0 : n[e]);
    }
    // immediate elements (past the cut-off): y = x.  Same operation sequence
    // as seed<T, n> + the recursion (+ the upward ladder in fp64).
    {
      const int wmax = __reduce_max_sync(kFull, (unsigned)wmax_l);
      const int bits = 32 - __clz(wmax | 1);
      T r[EPL], sr[EPL], xr[EPL];
      // everything still needed of x and n (deferred elements: a harmless 1/x
      // operand, so x = 0 in the queue does not send the warp to the cold
      // path, and order 0: no recursion steps, their values are never used)
      int neff[EPL];
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        xr[e] = wr[e] ? x[e] : T(1);
        tx[e] = A::add(x[e], x[e]);
        neff[e] = wr[e] ? n[e] : 0;
      }
      // correctly rounded 1/x and sqrt through their branch-free fast paths
      // (bit-identical to the intrinsics)
      bool slow = false;
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        bool sj;
        r[e] = A::rcp_fast(xr[e], sj);
        slow = slow || sj;
      }
      if (__any_sync(kFull, slow)) {
#pragma unroll
        for (int e = 0; e < EPL; ++e) r[e] = A::rcp_cold(xr[e]);
      }
      slow = false;
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        bool sj;
        sr[e] = A::sqrt_fast(r[e], sj);
        slow = slow || sj;
      }
      if (__any_sync(kFull, slow)) {
#pragma unroll
        for (int e = 0; e < EPL; ++e) sr[e] = A::sqrt_cold(r[e]);
      }
      // r^n, bit by bit over all elements (powi_rt_bounded's product sequence)
      T pw[EPL], pp[EPL];
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        pw[e] = (neff[e] & 1) ? r[e] : T(1);
        pp[e] = r[e];
      }
#pragma unroll
      for (int j = 1; j < 5; ++j) {
        if (j >= bits) break;
#pragma unroll
        for (int e = 0; e < EPL; ++e) pp[e] = A::mul(pp[e], pp[e]);
#pragma unroll
        for (int e = 0; e < EPL; ++e) pw[e] = A::mul(pw[e], ((neff[e] >> j) & 1) ? pp[e] : T(1));
      }
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        // n = 0: the power is exactly 1.0 and (c * 1.0) * sr == c * sr, so no select
        cur[e] = A::mul(A::mul(zc[e].c, pw[e]), sr[e]);
      }
#pragma unroll
      for (int e = 0; e < EPL; ++e)
        if (wr[e]) dst[e][neff[e]] = cur[e];
      // recursion steps m = wmax-1 .. 0: enter the unrolled chain once through
      // a jump table (wmax is warp-uniform) instead of testing every step
      // one predicate per element and step: elements that are not written
      // here (deferred, padding) take no steps (their cur is never used)
      if (!kTwoSets) advance();                  // x, n, goff are dead from here
#define BOYS_STEP(M)                                                       \
  if ((M) < NB) {                                                           \
    T nx[EPL];                                                              \
    _Pragma("unroll") for (int e = 0; e < EPL; ++e)                         \
      nx[e] = A::fma(tx[e], cur[e], t[e]);                                  \
    _Pragma("unroll") for (int e = 0; e < EPL; ++e)                         \
      nx[e] = A::mul(nx[e], rinv<T>((M) < NB ? (M) : 0));                   \
    _Pragma("unroll") for (int e = 0; e < EPL; ++e)                         \
      pmov((M) < neff[e], cur[e], nx[e]);                                   \
    _Pragma("unroll") for (int e = 0; e < EPL; ++e)                         \
      psts((M) < neff[e], dst[e] + (M), cur[e]);                            \
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
    }
    __syncwarp();
    // the chunk's output range [base, base + cnt): scalar head/tail to reach
    // 16-byte alignment, one bulk async copy (TMA engine) for the body
    // (16-byte vector stores by all lanes instead: 1.55 vs 1.42 ms f64, 0.81 vs
    // 0.76 ms f32).
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
        // operands through warp reductions (identical on every lane): they
        // land in uniform registers, which the bulk-copy instruction takes,
        // without the vector-to-uniform waterfall loop
        const uintptr_t g = reinterpret_cast<uintptr_t>(out + base + head);
        const unsigned glo = __reduce_max_sync(kFull, (unsigned)g);
        const unsigned ghi = __reduce_max_sync(kFull, (unsigned)(g >> 32));
        const unsigned sa = __reduce_max_sync(kFull, smem_u32(W.stage + shift + head));
        const unsigned nb = __reduce_max_sync(kFull, (unsigned)(body * sizeof(T)));
        if (lane == 0) bulk_store_u(((uint64_t)ghi << 32) | glo, sa, nb);
      }
    }
    while (qn >= 32) qn = ragged_drain<T, NB>(W, rows, qn, out);
  }
  while (qn > 0) qn = ragged_drain<T, NB>(W, rows, qn, out);
  if (lane == 0) bulk_wait_all();
  // the batch's last, partial chunk: per element, by the warp whose sequence
  // of chunks reaches it
  if (c == nfull && nfull * CH < N) {
#pragma unroll 1
    for (int e = 0; e < EPL; ++e) {
      const int64_t j = nfull * CH + 32 * e + lane;
      const bool jin = j < N;
      ragged_general_element<T>(jin ? ldg_nc(X + j) : T(0), jin ? (int)NM[j] : 0,
                                jin ? __ldg(OFF + j) : 0, jin, j, out, dom);
    }
  }
}

// (A block-window ragged variant -- 1024-element windows counting-sorted into
// order buckets, one compile-time-order tail per warp task -- measured slower
// than the warp chunks for both dtypes (f64 2.59 vs 1.92 ms, f32 1.19 vs
// 1.00 ms) and was removed; it is in the history up to commit 50d605b.)

// ---------------------------------------------------------------------------
// ragged offsets: exclusive prefix sum of (n_i + 1), O(N), no workspace.  The
// output array itself parks the nblk tile totals R and the ngrp group sums GS
// contiguously at its tail (GS, R = OFF[N + 1 - ngrp - nblk .. N], inside the
// last few tiles):
//   1. block b sums its tiles' orders and stores R[b] (coalesced, 4 tiles per
//      block, all loads in flight);
//   2. block g scans R[1024 g ..] in place (exclusive, within the group) and
//      parks the group's sum GS[g] just before R;
//   3. block b < tfirst takes R[b] + sum(GS[< b/1024]) and scans its tile from
//      it (shared-memory transpose, so the int64 stores leave coalesced);
//      tiles tfirst.. overlap the parked words and are left to
//   4. one block that first reads their prefixes, then writes those tiles and
//      OFF[N] (the grand total).
// Traffic: n_max read twice + offsets written once (~1.21 GB at 2^27).
// ---------------------------------------------------------------------------
constexpr int kScanPer = 16;                         // elements per thread
constexpr int kScanTile = kThreads * kScanPer;       // 4096 elements per tile
constexpr int kTotTiles = 4;                         // tiles per totals block

// the thread's 16 consecutive orders (16-byte vector load when aligned)
__device__ __forceinline__ void scan_load16(const uint8_t* __restrict__ NM, int64_t N, int64_t i0,
                                            bool vec, int (&v)[kScanPer]) {
  if (vec && i0 + kScanPer <= N) {
    const uint4 q = __ldg(reinterpret_cast<const uint4*>(NM + i0));
    const unsigned w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) v[k] = (int)((w[k >> 2] >> (8 * (k & 3))) & 0xffu) + 1;
  } else {
#pragma unroll
    for (int k = 0; k < kScanPer; ++k) v[k] = (i0 + k < N) ? (int)NM[i0 + k] + 1 : 0;
  }
}

// sum of (n + 1) over 16 consecutive orders (SIMD byte sums when aligned)
__device__ __forceinline__ int scan_sum16(const uint8_t* __restrict__ NM, int64_t N, int64_t i0,
                                          bool vec) {
  if (vec && i0 + kScanPer <= N) {
    const uint4 q = __ldg(reinterpret_cast<const uint4*>(NM + i0));
    // __vsadu4(w, 0): sum of the 4 bytes of w
    return (int)(__vsadu4(q.x, 0u) + __vsadu4(q.y, 0u) + __vsadu4(q.z, 0u) + __vsadu4(q.w, 0u)) +
           kScanPer;
  }
  int s = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) s += (i0 + k < N) ? (int)NM[i0 + k] + 1 : 0;
  return s;
}

// block-wide exclusive scan of one int64 per thread (warp shuffles + 8 warp sums)
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* s_warp, int64_t& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int64_t o = __shfl_up_sync(kFull, inc, d);
    if (lane >= d) inc += o;
  }
  if (lane == 31) s_warp[wid] = inc;
  __syncthreads();
  int64_t wpre = 0;
  total = 0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) {
    const int64_t t = s_warp[w];
    wpre += w < wid ? t : 0;
    total += t;
  }
  return wpre + inc - v;
}

__global__ void __launch_bounds__(kThreads)
offsets_totals_kernel(const uint8_t* __restrict__ NM, int64_t N, int32_t* __restrict__ R,
                      int64_t nblk, bool vec) {
  __shared__ int s_warp[kTotTiles][kThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int sum[kTotTiles];
#pragma unroll
  for (int q = 0; q < kTotTiles; ++q) {       // loads of the block's tiles all in flight
    const int64_t b = (int64_t)blockIdx.x * kTotTiles + q;
    sum[q] = b < nblk ? scan_sum16(NM, N, b * kScanTile + (int64_t)threadIdx.x * kScanPer, vec) : 0;
  }
#pragma unroll
  for (int q = 0; q < kTotTiles; ++q) {
    const int s = __reduce_add_sync(kFull, (unsigned)sum[q]);
    if (lane == 0) s_warp[q][wid] = s;
  }
  __syncthreads();
  if (threadIdx.x < kTotTiles) {
    const int q = threadIdx.x;
    const int64_t b = (int64_t)blockIdx.x * kTotTiles + q;
    int t = 0;                               // <= 4096 * 256: int32
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) t += s_warp[q][w];
    if (b < nblk) R[b] = t;
  }
}

// group g (1024 totals, one per thread): R[g*1024 ..] <- exclusive prefix
// sums within the group, in place; GS[g] <- the group's sum
__global__ void __launch_bounds__(1024)
offsets_groups_kernel(int64_t nblk, int32_t* __restrict__ R, int64_t* __restrict__ GS) {
  __shared__ int64_t s_warp[32];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int64_t b = (int64_t)blockIdx.x * 1024 + t;
  const int64_t v = b < nblk ? (int64_t)R[b] : 0;
  int64_t inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int64_t o = __shfl_up_sync(kFull, inc, d);
    if (lane >= d) inc += o;
  }
  if (lane == 31) s_warp[wid] = inc;
  __syncthreads();
  int64_t wpre = 0, total = 0;
#pragma unroll 8
  for (int w = 0; w < 32; ++w) {
    const int64_t sw = s_warp[w];
    wpre += w < wid ? sw : 0;
    total += sw;
  }
  if (b < nblk) R[b] = (int32_t)(wpre + inc - v);    // in-group prefix < 2^31
  if (t == 0) GS[blockIdx.x] = total;
}

// exclusive prefix of tile b: its in-group prefix + the sums of the groups
// before it (one warp; every lane returns it)
__device__ __forceinline__ int64_t tile_prefix(const int32_t* __restrict__ R,
                                               const int64_t* __restrict__ GS, int64_t b) {
  const int lane = threadIdx.x & 31;
  const int64_t g = b >> 10;
  int64_t acc = 0;
  for (int64_t q = lane; q < g; q += 32) acc += GS[q];
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) acc += __shfl_xor_sync(kFull, acc, d);
  return acc + R[b];
}

// one tile (kScanTile orders from b0) scanned from `prefix` and written to OFF
// (256 threads; shared-memory transpose so the int64 stores leave coalesced).
// Returns the tile's total on every thread.
// The prefix comes from get_prefix() (called by every thread after the tile's
// loads are issued; it must publish to *s_pre from one thread), read after the
// block scan's barrier, so its loads overlap the tile's.
template <typename GetPrefix>
__device__ __forceinline__ int64_t scan_write_tile(const uint8_t* __restrict__ NM, int64_t N,
                                                   int64_t* __restrict__ OFF, int64_t b0,
                                                   GetPrefix&& get_prefix, int64_t* s_pre,
                                                   bool vec, int64_t* s_warp, int64_t* s_out) {
  constexpr int RS = kScanPer + 1;           // padded row: conflict-free row writes
  const int t = threadIdx.x & (kThreads - 1);
  int v[kScanPer];
  scan_load16(NM, N, b0 + (int64_t)t * kScanPer, vec, v);
  get_prefix();
  int sum = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) sum += v[k];
  int64_t total;
  const int64_t local = block_excl_scan(sum, s_warp, total);
  int64_t p = *s_pre + local;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    s_out[t * RS + k] = p;
    p += v[k];
  }
  __syncthreads();
  const int cnt = (int)min((int64_t)kScanTile, N - b0);
  for (int k = t; k < cnt; k += kThreads)
    OFF[b0 + k] = s_out[(k / kScanPer) * RS + (k % kScanPer)];
  __syncthreads();                           // s_warp / s_out reuse
  return total;
}

__global__ void __launch_bounds__(kThreads)
offsets_tiles_kernel(const uint8_t* __restrict__ NM, int64_t N, int64_t* __restrict__ OFF,
                     const int32_t* __restrict__ R, const int64_t* __restrict__ GS, bool vec) {
  __shared__ int64_t s_warp[kThreads / 32];
  __shared__ int64_t s_out[kThreads * (kScanPer + 1)];
  __shared__ int64_t s_pre;
  const int64_t b = blockIdx.x;
  scan_write_tile(NM, N, OFF, b * kScanTile, [&] {
    if (threadIdx.x < 32) {
      const int64_t p = tile_prefix(R, GS, b);
      if (threadIdx.x == 0) s_pre = p;
    }
  }, &s_pre, vec, s_warp, s_out);
}

// tiles tfirst..nblk-1 (their outputs overlap R): prefixes first, then writes
__global__ void __launch_bounds__(kThreads)
offsets_tail_kernel(const uint8_t* __restrict__ NM, int64_t N, int64_t* __restrict__ OFF,
                    const int32_t* __restrict__ R, const int64_t* __restrict__ GS,
                    int64_t tfirst, int64_t nblk, bool vec) {
  extern __shared__ int64_t s_pre[];         // nblk - tfirst prefixes
  __shared__ int64_t s_warp[kThreads / 32];
  __shared__ int64_t s_out[kThreads * (kScanPer + 1)];
  const int wid = threadIdx.x >> 5;
  for (int64_t q = wid; q < nblk - tfirst; q += kThreads / 32) {
    const int64_t p = tile_prefix(R, GS, tfirst + q);
    if ((threadIdx.x & 31) == 0) s_pre[q] = p;
  }
  __syncthreads();
  int64_t last = 0;
  for (int64_t b = tfirst; b < nblk; ++b)
    last = s_pre[b - tfirst] + scan_write_tile(NM, N, OFF, b * kScanTile, [] {}, &s_pre[b - tfirst],
                                               vec, s_warp, s_out);
  if (threadIdx.x == 0) OFF[N] = last;       // grand total
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
    // Same-box A/Bs on cfg4 (tools/ragged_rate.py), current kernel:
    //  * elements per lane: 3 (f64; 2: 1.64-1.70 vs 1.50 ms, also with three
    //    resident blocks) and 4 (f32; 3: 0.77-0.78 vs 0.75 ms; 4 with four
    //    resident blocks spills: 0.95 ms);
    //  * 12 staged values per element; 256-thread blocks (f64 192 threads x 3
    //    blocks: 1.59 ms, 128 x 4: 1.50 ms vs 1.43 ms); f64 at three resident
    //    blocks (8 staged values, 80 registers, spills): 1.65-1.72 vs 1.42 ms;
    //  * f64 recursion aligned at the chain start (no select on `cur`; the
    //    per-lane RN(1/(2M+1)) from shared memory one step ahead): ptxas copies
    //    the prefetched multipliers at every jump-table label (6 moves per
    //    step that wait on the loads): 1.67 vs 1.42 ms;
    //  * the chunk loop unrolled by two (no register copies between the two
    //    sets; 120 registers, twice the code): 1.75 vs 1.42 ms;
    //  * order-sorted rounds were costed from the profile and not built: the
    //    recursion is 6 instructions per element and step, a single-slot step
    //    costs ~11 with its loop, so sorting 96 elements buys less than its
    //    ballots and shared-memory permutation cost.
#ifndef BOYS_AB_EPL64
#define BOYS_AB_EPL64 3
#endif
#ifndef BOYS_AB_EPL32
#define BOYS_AB_EPL32 4
#endif
#ifndef BOYS_AB_CPE
#define BOYS_AB_CPE 12
#endif
    constexpr int EPL = sizeof(T) == 8 ? BOYS_AB_EPL64 : BOYS_AB_EPL32, CPE = BOYS_AB_CPE;
    boys_status st = launch_chunks<T, NB, EPL, CPE, 0>(x, nm, off, N, out, dom, s);
    if (st != BOYS_OK) return st;
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_status(cudaGetLastError());
}

boys_status eval_ragged_base(boys_dtype dtype, const void* x, const uint8_t* nm,
                             const int64_t* off, int64_t N, void* out, int64_t* dom,
                             cudaStream_t s) {
  if (dtype == BOYS_F64) return launch_ragged<double>(x, nm, off, N, out, dom, s);
  return launch_ragged<float>(x, nm, off, N, out, dom, s);
}

boys_status ragged_offsets_base(const uint8_t* nmax_dev, int64_t N, int64_t* offsets_dev,
                                cudaStream_t s) {
  if (N == 0) return cuda_status(cudaMemsetAsync(offsets_dev, 0, sizeof(int64_t), s));
  const int64_t nblk = (N + kScanTile - 1) / kScanTile;
  const int64_t ngrp = (nblk + 1023) / 1024;
  if (nblk > INT32_MAX) return BOYS_E_ARG;
  const bool vec = (reinterpret_cast<uintptr_t>(nmax_dev) & 15) == 0;
  // parked at the array's tail: group sums GS (int64), then the tile totals R
  // (int32: a tile's total is at most 4096 * 256)
  const int64_t park = ngrp + (nblk + 1) / 2;            // int64 words, <= N + 1
  int64_t* GS = offsets_dev + (N + 1 - park);
  int32_t* R = reinterpret_cast<int32_t*>(GS + ngrp);
  // first tile overlapping the parked words (at least the last tile: it also writes OFF[N])
  const int64_t tfirst = min((N + 1 - park) / kScanTile, nblk - 1);
  const int64_t ntail = nblk - tfirst;
  if (ntail * (int64_t)sizeof(int64_t) > 12 * 1024) return BOYS_E_ARG;    // N > ~2^33
  offsets_totals_kernel<<<(unsigned)((nblk + kTotTiles - 1) / kTotTiles), kThreads, 0, s>>>(
      nmax_dev, N, R, nblk, vec);
  offsets_groups_kernel<<<(unsigned)ngrp, 1024, 0, s>>>(nblk, R, GS);
  int launches = 3;
  if (tfirst > 0) {
    offsets_tiles_kernel<<<(unsigned)tfirst, kThreads, 0, s>>>(nmax_dev, N, offsets_dev, R, GS,
                                                                vec);
    ++launches;
  }
  offsets_tail_kernel<<<1, kThreads, ntail * sizeof(int64_t), s>>>(nmax_dev, N, offsets_dev, R,
                                                                     GS, tfirst, nblk, vec);
  g_launches.fetch_add(launches, std::memory_order_relaxed);
  return cuda_status(cudaGetLastError());
}

}  // namespace boys
