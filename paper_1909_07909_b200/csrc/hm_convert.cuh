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

#include "hm_fast.cuh"

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

// DMMA version, one pass over all levels (leaf b a multiple of 64, k in
// {16, 32, 64}): a CTA owns 64 rows (8 warps x 8 rows, inside one node on every
// level); a warp keeps its rows of U^(l) and V^(l) in registers in the DMMA
// accumulator layout and, level by level, writes U_l = U^(l) S, V_l = V^(l) and
// moves on to U^(l-1) = U^(l) R_ch, V^(l-1) = V^(l) W_ch. The accumulator
// fragment of one product is the A fragment of the next: lane (i, j) holds
// columns 8t + 2j + e of row i, so contraction chunk (t, e) is the k-index set
// {8t + e, 8t + 2 + e, 8t + 4 + e, 8t + 6 + e} (a permutation of the sum), and
// the B fragment reads matrix rows 8t + 2j + e (shared memory, row stride
// KT + 2: conflict-free). S, R_ch, W_ch of the level's node are staged per CTA.
// U and V are read once, every output written once: bytes = 8 (2 n k + 2 p n k).
template <int KT>
__device__ __forceinline__ void conv_prod(double (&out)[KT / 8][2], const double (&a)[KT / 8][2], const double* Bs,
                                          int lane) {
  constexpr int NT = KT / 8, ZB = KT + 2;
  const int i = lane >> 2, j = lane & 3;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) out[nt][0] = out[nt][1] = 0.0;
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const double* br = Bs + (8 * t + 2 * j + e) * ZB + i;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) dmma(out[nt][0], out[nt][1], a[t][e], br[8 * nt]);
    }
}

template <int KT>
__global__ void __launch_bounds__(256) hss2hodlr_mma_kernel(const ConvertParams P) {
  constexpr int NT = KT / 8, ZB = KT + 2;
  extern __shared__ __align__(16) double cbs[];  // [3][KT][ZB]: S, R_ch, W_ch of the CTA's node
  double* bs[3] = {cbs, cbs + KT * ZB, cbs + 2 * KT * ZB};
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = lane >> 2, j = lane & 3;
  const int64_t n = P.n, nk = n * KT;
  const int64_t rc = (int64_t)blockIdx.x * 64;      // the CTA's first row
  const int64_t row = rc + 8 * warp + i;            // this lane's row
  double u[NT][2], v[NT][2], t0[NT][2], t1[NT][2];
  {
    const double* Up = P.Uh + (int64_t)(P.p - 1) * nk + row * KT;  // leaf bases, copied in by the host
    const double* Vp = P.Vh + (int64_t)(P.p - 1) * nk + row * KT;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const double2 a = *reinterpret_cast<const double2*>(Up + 8 * t + 2 * j);
      const double2 c = *reinterpret_cast<const double2*>(Vp + 8 * t + 2 * j);
      u[t][0] = a.x; u[t][1] = a.y;
      v[t][0] = c.x; v[t][1] = c.y;
    }
  }
  for (int l = P.p; l >= 1; --l) {
    const int64_t a = rc / (P.b << (P.p - l));  // level-l node of the CTA's rows
    const int64_t q = a >> 1;
    const int w = (int)(a & 1);
    const double* S = P.B + ((((int64_t)1 << (l - 1)) - 1 + q) * 2 + w) * KT * KT;
    const double* Rh = l >= 2 ? P.R + ((((int64_t)1 << (l - 1)) - 2 + q) * 2 + w) * KT * KT : nullptr;
    const double* Wh = l >= 2 ? P.W + ((((int64_t)1 << (l - 1)) - 2 + q) * 2 + w) * KT * KT : nullptr;
    __syncthreads();  // previous level's fragments consumed
    for (int e = threadIdx.x; e < KT * KT / 2; e += blockDim.x) {
      const int r = e / (KT / 2), c = (e % (KT / 2)) * 2;
      cp_async16(&bs[0][r * ZB + c], S + r * KT + c);
      if (Rh) {
        cp_async16(&bs[1][r * ZB + c], Rh + r * KT + c);
        cp_async16(&bs[2][r * ZB + c], Wh + r * KT + c);
      }
    }
    cp_async_wait_all();
    __syncthreads();
    conv_prod<KT>(t0, u, bs[0], lane);  // U_l rows = U^(l) S
    double* Ul = P.Uh + (int64_t)(l - 1) * nk + row * KT;
    double* Vl = P.Vh + (int64_t)(l - 1) * nk + row * KT;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      *reinterpret_cast<double2*>(Ul + 8 * t + 2 * j) = make_double2(t0[t][0], t0[t][1]);
      if (l < P.p) *reinterpret_cast<double2*>(Vl + 8 * t + 2 * j) = make_double2(v[t][0], v[t][1]);  // V_l = V^(l)
    }
    if (l >= 2) {
      conv_prod<KT>(t0, u, bs[1], lane);  // U^(l-1) = U^(l) R_ch
      conv_prod<KT>(t1, v, bs[2], lane);  // V^(l-1) = V^(l) W_ch
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        u[t][0] = t0[t][0]; u[t][1] = t0[t][1];
        v[t][0] = t1[t][0]; v[t][1] = t1[t][1];
      }
    }
  }
}

}  // namespace hm
