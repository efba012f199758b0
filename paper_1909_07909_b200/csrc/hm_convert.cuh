// hm_convert.cuh — hss2hodlr on the GPU ("hss2hodlr ...
// by simply building explicit low-rank factorizations").
//
// The level-l bases of eq. (3) are built level by level from the
// leaves: U^(p) = U, and rows of child ch of node (l-1, i) get
//   U^(l-1) = U^(l) R_{U,i}^(l-1)[ch],   V^(l-1) = V^(l) W_{i}^(l-1)[ch].
// The HODLR factors of level l (Def. 2.2) are then
//   U_l(I_a) = U_a^(l) S_{a, sib a}  (S = B12 for a = 2q, B21 for a = 2q+1),
//   V_l(I_b) = V_b^(l).
// One launch per level l = p..1, in place in the output: level l of Uh holds
// U^(l) on entry (the leaf bases copied in for l = p, written by the level-l+1
// launch otherwise) and U_l on exit; level l of Vh holds V^(l) = V_l. Each CTA
// owns a tile of rows: it stages their U^(l), V^(l) rows in shared memory,
// then writes U_l, U^(l-1), V^(l-1) for them (row-local: no inter-CTA hazard).
// Fixed-order sums: bitwise repeatable.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hm {

struct ConvertParams {
  const double* R;  // [2^p-2][2k][k]
  const double* W;
  const double* B;  // [2^p-1][2][k][k]
  double* Uh;       // [p][n][k]
  double* Vh;
  int64_t n, b;
  int32_t p, k;
};

constexpr int kConvRows = 32;  // rows per CTA tile

__global__ void __launch_bounds__(256) hss2hodlr_level_kernel(const ConvertParams P, int l) {
  extern __shared__ double cs[];
  const int k = P.k;
  const int64_t n = P.n;
  const int64_t r0 = (int64_t)blockIdx.x * kConvRows;
  const int rows = (int)(n - r0 < kConvRows ? n - r0 : kConvRows);
  double* Ul = P.Uh + (int64_t)(l - 1) * n * k;
  double* Vl = P.Vh + (int64_t)(l - 1) * n * k;
  double* us = cs;                    // [rows][k]: U^(l)
  double* vs = cs + kConvRows * k;    // [rows][k]: V^(l)
  for (int e = threadIdx.x; e < rows * k; e += blockDim.x) {
    us[e] = Ul[r0 * k + e];
    vs[e] = Vl[r0 * k + e];
  }
  __syncthreads();
  const int64_t s_l = P.b << (P.p - l);  // rows per level-l node
  for (int o = threadIdx.x; o < rows * k; o += blockDim.x) {
    const int r = o / k, e = o - r * k;
    const int64_t row = r0 + r;
    const int64_t a = row / s_l;  // level-l node of the row
    const double* S = P.B + ((((int64_t)1 << (l - 1)) - 1 + (a >> 1)) * 2 + (a & 1)) * k * k;
    const double* u = us + r * k;
    double acc = 0.0;
    for (int f = 0; f < k; ++f) acc = fma(u[f], __ldg(S + f * k + e), acc);
    if (l >= 2) {
      const int64_t node = ((int64_t)1 << (l - 1)) - 2 + (a >> 1);  // parent (l-1, a>>1)
      const double* Rh = P.R + (node * 2 + (a & 1)) * k * k;
      const double* Wh = P.W + (node * 2 + (a & 1)) * k * k;
      const double* v = vs + r * k;
      double au = 0.0, av = 0.0;
      for (int f = 0; f < k; ++f) {
        au = fma(u[f], __ldg(Rh + f * k + e), au);
        av = fma(v[f], __ldg(Wh + f * k + e), av);
      }
      P.Uh[(int64_t)(l - 2) * n * k + row * k + e] = au;
      P.Vh[(int64_t)(l - 2) * n * k + row * k + e] = av;
    }
    Ul[row * k + e] = acc;
  }
}

}  // namespace hm
