// hm_treegemv.cuh — HSS tree levels for few right-hand sides (nrhs <= 4), where
// every node operation is a matrix-vector product and the levels are bound by
// streaming the generators W, R, B from HBM:
//
//   upsweep   x_l[i]    = W_{l,i}^T [x_{l+1}[2i]; x_{l+1}[2i+1]]
//   down      y_l[2q+w] = S_w x_l[2q+1-w] + R_{l-1,q}[w] y_{l-1}[q]       (G1)
//
// One warp per node, no shared memory, no block barrier; every generator row
// is read by 128-bit loads with many independent loads in flight per lane.
// Upsweep: lanes own output columns a (K = 32: one each; K = 64: two; K = 16:
// two half-warps take alternate rows and are added at the end), the children's
// coefficients are broadcast from registers with shuffles. Downsweep: lanes
// own output rows a and read their row of S (and of R_w) as 128-bit loads;
// x and y_parent broadcast by shuffles; for K = 16 the two half-warps split
// the contraction range and are added with one shuffle. Fixed summation order:
// bitwise repeatable. The top levels (few nodes) run in one cooperative launch
// with a grid barrier between levels (hss_tree_gemv_sweep_kernel).
#pragma once
#include <cooperative_groups.h>

#include "hm_fast.cuh"

namespace hm {

struct TreeGemvParams {
  const double* W;   // [2^p-2][2k][k]
  const double* R;   // [2^p-2][2k][k]
  const double* B;   // [2^p-1][2][k][k]
  double* xh;        // level-major [.][k][m]
  double* yh;
  const double* R_root;  // distributed subtree: translation of the subtree root [2k][k] (level-1 term)
  const double* y_root;  //                       and its y block [k][m]
  int32_t m;             // nrhs <= MB
  int32_t bt;            // 1: adjoint cores S'_w = B[1-w]^T
};

__device__ __forceinline__ double shfl(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
// keep a batch of loads in flight: every value must be available here (see reg_fence)
__device__ __forceinline__ void reg_fence1(double& v) { asm volatile("" : "+d"(v)); }

// value z[r][c] of a [rows][m] block held one row per lane (lane r % 32, slot r / 32)
template <int NS, int MB>
__device__ __forceinline__ double bcast(const double (&z)[NS][MB], int r, int c) {
  double v = z[0][c];
#pragma unroll
  for (int s = 1; s < NS; ++s)
    if ((r >> 5) == s) v = z[s][c];
  return shfl(v, r & 31);
}

// x_l[i] for one node (warp), K = rank, MB >= m.
template <int K, int MB, bool COH>
__device__ __forceinline__ void gemv_up_node(const TreeGemvParams& P, int l, int64_t i, int lane) {
  const int m = P.m;
  const int64_t km = (int64_t)K * m;
  const double* Wn = P.W + (((int64_t)1 << l) - 2 + i) * 2 * K * K;
  const double* z = P.xh + (((int64_t)1 << (l + 1)) - 2 + 2 * i) * km;  // [2K][m], children contiguous
  constexpr int NS = (2 * K + 31) / 32;
  double zr[NS][MB];
#pragma unroll
  for (int s = 0; s < NS; ++s)
#pragma unroll
    for (int c = 0; c < MB; ++c) {
      const int r = 32 * s + lane;
      zr[s][c] = (r < 2 * K && c < m) ? ld_operand<COH>(z + (int64_t)r * m + c) : 0.0;
    }
  double* out = P.xh + (((int64_t)1 << l) - 2 + i) * km;
  if constexpr (K == 32) {
    double acc[MB] = {};
    constexpr int U = 2 * K;  // every row of W in flight at once (latency of small levels)
#pragma unroll 1
    for (int r0 = 0; r0 < 2 * K; r0 += U) {
      double w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) w[u] = ldg_stream(Wn + (r0 + u) * K + lane);
#pragma unroll
      for (int u = 0; u < U; ++u) reg_fence1(w[u]);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int c = 0; c < MB; ++c) acc[c] = fma(w[u], bcast<NS, MB>(zr, r0 + u, c), acc[c]);
    }
#pragma unroll
    for (int c = 0; c < MB; ++c)
      if (c < m) out[lane * m + c] = acc[c];
  } else if constexpr (K == 64) {
    double acc[2][MB] = {};
    constexpr int U = 32;
#pragma unroll 1
    for (int r0 = 0; r0 < 2 * K; r0 += U) {
      double2 w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) w[u] = ldg_stream2(Wn + (r0 + u) * K + 2 * lane);
#pragma unroll
      for (int u = 0; u < U; ++u) reg_fence(w[u]);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int c = 0; c < MB; ++c) {
          const double zz = bcast<NS, MB>(zr, r0 + u, c);
          acc[0][c] = fma(w[u].x, zz, acc[0][c]);
          acc[1][c] = fma(w[u].y, zz, acc[1][c]);
        }
    }
#pragma unroll
    for (int c = 0; c < MB; ++c)
      if (c < m) {
        out[(2 * lane) * m + c] = acc[0][c];
        out[(2 * lane + 1) * m + c] = acc[1][c];
      }
  } else {  // K == 16: half-warp h takes rows r = 2 t + h; halves added at the end
    const int a = lane & 15, h = lane >> 4;
    double acc[MB] = {};
    constexpr int U = K;
#pragma unroll 1
    for (int t0 = 0; t0 < K; t0 += U) {
      double w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) w[u] = ldg_stream(Wn + (2 * (t0 + u) + h) * K + a);
#pragma unroll
      for (int u = 0; u < U; ++u) reg_fence1(w[u]);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int c = 0; c < MB; ++c) {
          // both halves need z rows 2t and 2t+1: broadcast both, select
          const double z0 = bcast<NS, MB>(zr, 2 * (t0 + u), c), z1 = bcast<NS, MB>(zr, 2 * (t0 + u) + 1, c);
          acc[c] = fma(w[u], h ? z1 : z0, acc[c]);
        }
    }
#pragma unroll
    for (int c = 0; c < MB; ++c) {
      const double other = __shfl_down_sync(0xffffffffu, acc[c], 16);
      if (h == 0 && c < m) out[a * m + c] = acc[c] + other;
    }
  }
}

// y_l[j] for one node (warp).
template <int K, int MB, bool COH>
__device__ __forceinline__ void gemv_down_node(const TreeGemvParams& P, int l, int64_t j, int lane) {
  const int m = P.m;
  const int64_t km = (int64_t)K * m;
  const int64_t q = j >> 1;
  const int w = (int)(j & 1);
  const bool adj = P.bt != 0;
  const double* S = P.B + ((((int64_t)1 << (l - 1)) - 1 + q) * 2 + (adj ? 1 - w : w)) * K * K;
  const double* Rw = (l >= 2) ? P.R + ((((int64_t)1 << (l - 1)) - 2 + q) * 2 * K + (int64_t)w * K) * K
                              : (P.R_root ? P.R_root + (int64_t)w * K * K : nullptr);
  const double* xs = P.xh + (((int64_t)1 << l) - 2 + (j ^ 1)) * km;
  const double* yp = (l >= 2) ? P.yh + (((int64_t)1 << (l - 1)) - 2 + q) * km : P.y_root;
  constexpr int NS = (K + 31) / 32;
  double xr[NS][MB], yr[NS][MB];
#pragma unroll
  for (int s = 0; s < NS; ++s)
#pragma unroll
    for (int c = 0; c < MB; ++c) {
      const int r = 32 * s + lane;
      xr[s][c] = (r < K && c < m) ? ld_operand<COH>(xs + (int64_t)r * m + c) : 0.0;
      yr[s][c] = (Rw && r < K && c < m) ? ld_operand<COH>(yp + (int64_t)r * m + c) : 0.0;
    }
  double* out = P.yh + (((int64_t)1 << l) - 2 + j) * km;
  // Lanes own output rows: K = 32: row lane; K = 64: rows lane, lane + 32;
  // K = 16: row lane & 15, and the two half-warps split the contraction range
  // (h = lane >> 4 takes r in [8h, 8h + 8)), added with one shuffle at the end.
  // Control flow is warp-uniform (every lane runs every shuffle).
  constexpr int RPL = K == 64 ? 2 : 1;
  constexpr int RL = K == 16 ? 8 : K;  // contraction length per lane
  const int h = K == 16 ? lane >> 4 : 0;
  const int rb = h * RL;
#pragma unroll
  for (int rr = 0; rr < RPL; ++rr) {
    const int a = K == 16 ? (lane & 15) : lane + 32 * rr;
    double acc[MB] = {};
    // S term: (S x)[a] = sum_r S[a][r] x[r]; adjoint: (S^T x)[a] = sum_r S[r][a] x[r];
    // then the R term (R_w y)[a]. Chunks of 8 contraction indices: 8 loads in
    // flight per lane before the FMAs.
    constexpr int CH = RL <= 32 ? RL : 16;  // contraction indices in flight per load batch
#pragma unroll 1
    for (int t0 = 0; t0 < RL; t0 += CH) {
      double sv[CH];
      if (!adj) {
#pragma unroll
        for (int t = 0; t < CH; t += 2) {
          const double2 v = ldg_stream2(S + (int64_t)a * K + rb + t0 + t);
          sv[t] = v.x;
          sv[t + 1] = v.y;
        }
      } else {
#pragma unroll
        for (int t = 0; t < CH; ++t) sv[t] = ldg_stream(S + (int64_t)(rb + t0 + t) * K + a);
      }
#pragma unroll
      for (int t = 0; t < CH; ++t) reg_fence1(sv[t]);
#pragma unroll
      for (int t = 0; t < CH; ++t)
#pragma unroll
        for (int c = 0; c < MB; ++c) acc[c] = fma(sv[t], bcast<NS, MB>(xr, rb + t0 + t, c), acc[c]);
    }
    if (Rw) {
#pragma unroll 1
      for (int t0 = 0; t0 < RL; t0 += CH) {
        double rv[CH];
#pragma unroll
        for (int t = 0; t < CH; t += 2) {
          const double2 v = ldg_stream2(Rw + (int64_t)a * K + rb + t0 + t);
          rv[t] = v.x;
          rv[t + 1] = v.y;
        }
#pragma unroll
        for (int t = 0; t < CH; ++t) reg_fence1(rv[t]);
#pragma unroll
        for (int t = 0; t < CH; ++t)
#pragma unroll
          for (int c = 0; c < MB; ++c) acc[c] = fma(rv[t], bcast<NS, MB>(yr, rb + t0 + t, c), acc[c]);
      }
    }
    if constexpr (K == 16) {
#pragma unroll
      for (int c = 0; c < MB; ++c) acc[c] += __shfl_down_sync(0xffffffffu, acc[c], 16);
    }
    if (K != 16 || h == 0)
#pragma unroll
      for (int c = 0; c < MB; ++c)
        if (c < m) out[(int64_t)a * m + c] = acc[c];
  }
}

template <int K, int MB>
__global__ void __launch_bounds__(256) hss_up_gemv_kernel(const TreeGemvParams P, int l) {
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (gw >= ((int64_t)1 << l)) return;
  gemv_up_node<K, MB, false>(P, l, gw, threadIdx.x & 31);
}

template <int K, int MB>
__global__ void __launch_bounds__(256) hss_down_gemv_kernel(const TreeGemvParams P, int l) {
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (gw >= ((int64_t)1 << l)) return;
  gemv_down_node<K, MB, false>(P, l, gw, threadIdx.x & 31);
}

// Levels up_from..1 (up) then 1..down_to (down) in one cooperative launch,
// warp per node, grid barrier between levels; .cg loads for in-launch data.
template <int K, int MB>
__global__ void __launch_bounds__(256) hss_tree_gemv_sweep_kernel(const TreeGemvParams P, int up_from, int down_to) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  bool first = true;
  for (int l = up_from; l >= 1; --l) {
    if (!first) grid.sync();
    first = false;
    for (int64_t i = gw; i < ((int64_t)1 << l); i += nw) gemv_up_node<K, MB, true>(P, l, i, lane);
  }
  for (int l = 1; l <= down_to; ++l) {
    if (!first) grid.sync();
    first = false;
    for (int64_t j = gw; j < ((int64_t)1 << l); j += nw) gemv_down_node<K, MB, true>(P, l, j, lane);
  }
}

}  // namespace hm
