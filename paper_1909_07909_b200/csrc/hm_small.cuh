// hm_small.cuh — the whole HSS product in ONE launch for small trees
// (BASELINE config 2: n = 4096, 64 leaves, 6 levels, k = 16, m = 16), where the
// cost is the dependency chain through the tree levels, not bytes or flops.
//
// Fig. 5 right with readings G1/G2, scheduled so that almost every
// dependent step stays inside one CTA (shared memory + __syncthreads, ~0.1 us)
// and only two steps cross CTAs (grid-wide barriers of the cooperative launch):
//   phase 1  CTA s < S owns the subtree of 2^h leaves under node (q, s), q = p-h:
//            Step 1 (x_i = V_i^T X(I_i)) for its leaves, upsweep to level q;
//            then signals `up`.
//   phase 2  CTA 0 waits for all S subtrees, runs the upsweep q-1..1 and the
//            coupling + downsweep for levels 1..q (every node), signals `top`.
//   phase 3  CTA c (one per leaf) waits for `top`, recomputes the coupling +
//            downsweep along its own root-to-leaf path for levels q+1..p (the
//            few ancestors inside its subtree; CTAs of sibling leaves write the
//            same ancestor blocks with bit-identical values, which is benign),
//            then Step 4 Y(I_c) = D_c X(I_c) + U_c y_c.
// The grid is launched cooperatively (all CTAs co-resident); the two hops are
// grid.sync() barriers. Data written in this launch is read with .cg loads
// (L2, coherent). Fixed-order sums: bitwise repeatable.
#pragma once
#include <cooperative_groups.h>

#include "hm_fast.cuh"

namespace hm {

struct SmallHssParams {
  const double *D, *U, *V, *R, *W, *B, *X;
  double* Y;
  double *xh, *yh;   // level-major coefficient blocks [.][k][m] (workspace)
  int32_t b, p, m, h;
  int32_t nsub;      // S = 2^(p-h)
  int32_t pad;
};

// Coefficient block of node (l, i) (l >= 1) in xh / yh.
__device__ __forceinline__ int64_t coef_off(int l, int64_t i, int64_t km) { return (((int64_t)1 << l) - 2 + i) * km; }

// Coupling + downsweep of node (l, j), rows 8 rg .. 8 rg + 7 (one warp):
// y_l[j] = S_w x_l[j^1] + (l >= 2 ? R_{l-1, j>>1}[w] y_{l-1}[j>>1] : 0), w = j & 1.
// yp: the parent's y block (ld m), global (COH) or null; out row-major ld m.
template <int KT, int NT>
__device__ __forceinline__ void small_down_rows(const SmallHssParams& P, int l, int64_t j, const double* yp, int rg,
                                                double* out, int lane) {
  const int m = P.m;
  const int64_t km = (int64_t)KT * m;
  const int64_t q = j >> 1;
  const int w = (int)(j & 1);
  const double* S = P.B + ((((int64_t)1 << (l - 1)) - 1 + q) * 2 + w) * KT * KT;
  double acc[1][NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) acc[0][nt][0] = acc[0][nt][1] = 0.0;
  warp_rowmajor_mma<1, NT, true, true, 2>(acc, S + (int64_t)8 * rg * KT, KT, KT, P.xh + coef_off(l, j ^ 1, km), m, m,
                                         lane);
  if (l >= 2) {
    const double* Rh = P.R + ((((int64_t)1 << (l - 1)) - 2 + q) * 2 * KT + (int64_t)w * KT) * KT;
    warp_rowmajor_mma<1, NT, true, true, 2>(acc, Rh + (int64_t)8 * rg * KT, KT, KT, yp, m, m, lane);
  }
  const int i = lane >> 2, jj = lane & 3;
  double* y = out + (int64_t)(8 * rg + i) * m;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int c = nt * 8 + 2 * jj;
    if (c < m) y[c] = acc[0][nt][0];
    if (c + 1 < m) y[c + 1] = acc[0][nt][1];
  }
}

template <int KT, int NT, int RG>
__global__ void __launch_bounds__(256) hss_small_kernel(const SmallHssParams P) {
  extern __shared__ __align__(16) double ssm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int p = P.p, h = P.h, q = p - h, m = P.m, b = P.b;
  const int64_t km = (int64_t)KT * m;
  // ---------------- phase 1: subtree Step 1 + upsweep to level q ----------------
  if (blockIdx.x < (unsigned)P.nsub) {
    const int64_t s = blockIdx.x;
    const int nl = 1 << h;
    for (int t = warp; t < nl * (KT / 16); t += 8) {  // leaves x (warp per rank group)
      const int64_t leaf = s * nl + t / (KT / 16);
      const int g = t % (KT / 16);
      double acc[2][NT][2];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[a][nt][0] = acc[a][nt][1] = 0.0;
      warp_transposed_mma<1, NT, false>(acc, P.V + leaf * b * KT + 16 * g, KT, P.X + leaf * b * m, m, 0, m, b, lane);
      store_transposed<1, NT>(acc, P.xh + coef_off(p, leaf, km) + (int64_t)16 * g * m, m, 0, m, lane);
    }
    for (int l = p - 1; l >= q && l >= 1; --l) {
      __syncthreads();  // level l+1 blocks of this subtree written (same CTA)
      const int cnt = 1 << (l - q);
      for (int t = warp; t < cnt * (KT / 16); t += 8) {
        const int64_t node = s * cnt + t / (KT / 16);
        const int g = t % (KT / 16);
        const double* Wn = P.W + (((int64_t)1 << l) - 2 + node) * 2 * KT * KT;
        double acc[2][NT][2];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) acc[a][nt][0] = acc[a][nt][1] = 0.0;
        warp_transposed_mma<1, NT, true>(acc, Wn + 16 * g, KT, P.xh + coef_off(l + 1, 2 * node, km), m, 0, m, 2 * KT,
                                         lane);
        store_transposed<1, NT>(acc, P.xh + coef_off(l, node, km) + (int64_t)16 * g * m, m, 0, m, lane);
      }
    }
  }
  cooperative_groups::this_grid().sync();  // every subtree's x blocks written
  // ---------------- phase 2: CTA 0, the top of the tree ----------------
  if (blockIdx.x == 0) {
    for (int l = q - 1; l >= 1; --l) {  // upsweep above the subtrees
      const int cnt = 1 << l;
      for (int t = warp; t < cnt * (KT / 16); t += 8) {
        const int64_t node = t / (KT / 16);
        const int g = t % (KT / 16);
        const double* Wn = P.W + (((int64_t)1 << l) - 2 + node) * 2 * KT * KT;
        double acc[2][NT][2];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) acc[a][nt][0] = acc[a][nt][1] = 0.0;
        warp_transposed_mma<1, NT, true>(acc, Wn + 16 * g, KT, P.xh + coef_off(l + 1, 2 * node, km), m, 0, m, 2 * KT,
                                         lane);
        store_transposed<1, NT>(acc, P.xh + coef_off(l, node, km) + (int64_t)16 * g * m, m, 0, m, lane);
      }
      __syncthreads();
    }
    for (int l = 1; l <= q; ++l) {  // coupling + downsweep, every node of levels 1..q
      const int cnt = 1 << l;
      for (int t = warp; t < cnt * (KT / 8); t += 8) {
        const int64_t j = t / (KT / 8);
        const int rg = t % (KT / 8);
        small_down_rows<KT, NT>(P, l, j, l >= 2 ? P.yh + coef_off(l - 1, j >> 1, km) : nullptr, rg,
                                P.yh + coef_off(l, j, km), lane);
      }
      __syncthreads();
    }
  }
  cooperative_groups::this_grid().sync();  // the top tree's y blocks written
  // ---------------- phase 3: per leaf, path downsweep q+1..p + Step 4 ----------------
  constexpr int MC = NT * 8, ZS = MC + 2;
  double* Zy = ssm;  // [KT][ZS]: y_leaf staged for the U product
  for (int64_t leaf = blockIdx.x; leaf < ((int64_t)1 << p); leaf += gridDim.x) {
    const double* yprev = q >= 1 ? P.yh + coef_off(q, leaf >> h, km) : nullptr;  // from phase 2 (global)
    for (int l = q + 1; l <= p; ++l) {
      const int64_t j = leaf >> (p - l);
      double* out = P.yh + coef_off(l, j, km);
      for (int rg = warp; rg < KT / 8; rg += 8) small_down_rows<KT, NT>(P, l, j, yprev, rg, out, lane);
      __threadfence_block();
      __syncthreads();
      yprev = out;
    }
    // Step 4: Y(I_leaf) = D_leaf X(I_leaf) + U_leaf y_leaf; warp w owns rows 8 RG w ..
    for (int e = threadIdx.x; e < KT * MC; e += blockDim.x) {
      const int r = e / MC, c = e - r * MC;
      Zy[r * ZS + c] = c < m ? ldg_cg(yprev + (int64_t)r * m + c) : 0.0;
    }
    __syncthreads();
    double acc[RG][NT][2];
#pragma unroll
    for (int rg = 0; rg < RG; ++rg)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[rg][nt][0] = acc[rg][nt][1] = 0.0;
    const int64_t r0 = leaf * b, wrow = (int64_t)warp * 8 * RG;
    warp_rowmajor_mma<RG, NT, true, false, 2>(acc, P.D + leaf * b * b + wrow * b, b, b, P.X + r0 * m, m, m, lane);
    warp_rowmajor_mma<RG, NT, false, false, 2>(acc, P.U + (r0 + wrow) * KT, KT, KT, Zy, ZS, MC, lane);
    const int i = lane >> 2, jj = lane & 3;
#pragma unroll
    for (int rg = 0; rg < RG; ++rg) {
      double* y = P.Y + (r0 + wrow + 8 * rg + i) * m;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int c = nt * 8 + 2 * jj;
        if (c < m) y[c] = acc[rg][nt][0];
        if (c + 1 < m) y[c + 1] = acc[rg][nt][1];
      }
    }
    __syncthreads();
  }
}

}  // namespace hm
