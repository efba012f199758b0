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

// ------------------------------------------------------------------ HODLR --
// The whole HODLR product for small problems (BASELINE config 1: n = 1024,
// 16 leaves, 4 levels) in ONE cooperative launch, CTA = leaf (Fig. 5 left,
// P:666-678, level-parallel as in the main path). Latency is the cost, so every
// input the CTA needs (D_L, the leaf's rows of every U_l and V_l, X(I_L)) is
// requested at once with cp.async at kernel start:
//   phase 1  partial t_l = V_l(I_L)^T X(I_L), every level, from shared memory,
//            to the workspace; grid-wide barrier.
//   phase 2  t_{l, sib(node_l(L))} = the sum of the partials of the 2^(p-l)
//            leaves under the sibling node, in leaf order (fixed: bitwise
//            repeatable); Y(I_L) = D_L X(I_L) + sum_l U_l(I_L) t_l from shared
//            memory, thread per output.
struct SmallHodlrParams {
  const double *D, *U, *V, *X;
  double* Y;
  double* part;       // [nleaves][ktot][m] partials
  int64_t n;
  int32_t b, p, m, ktot;
  int32_t k[kMaxLevels];   // ranks of levels 1..p (index l - 1)
  int64_t koff[kMaxLevels]; // sum of ranks of the levels before l (index l - 1)
};

// shared layout (doubles): D [b][b+2] | U [b][ktot] | V [b][ktot] | X [b][m] | T [ktot][m]
__host__ __device__ inline int64_t hodlr_small_smem_doubles(int64_t b, int64_t kt, int64_t m) {
  return b * (b + 2) + 2 * b * kt + b * m + kt * m + 8;
}

__global__ void __launch_bounds__(256) hodlr_small_kernel(const SmallHodlrParams P) {
  extern __shared__ __align__(16) double hsm[];
  const int64_t L = blockIdx.x, b = P.b, n = P.n;
  const int m = P.m, p = P.p, kt = P.ktot;
  const int64_t r0 = L * b;
  const int zd = (int)b + 2;
  double* Ds = hsm;
  double* Us = Ds + b * zd;
  double* Vs = Us + b * kt;
  double* Xs = Vs + b * kt;
  double* Ts = Xs + b * m;
  // every input of the CTA in flight at once
  stage_rows_async(Ds, zd, P.D + L * b * b, b, (int)b, (int)b, (int)b);
  {
    int64_t uoff = 0;
    for (int l = 1; l <= p; ++l) {
      const int k = P.k[l - 1];
      if (k > 0) {
        stage_rows_async(Us + P.koff[l - 1], kt, P.U + uoff + r0 * k, k, (int)b, k, k);
        stage_rows_async(Vs + P.koff[l - 1], kt, P.V + uoff + r0 * k, k, (int)b, k, k);
      }
      uoff += n * k;
    }
  }
  stage_rows_async(Xs, m, P.X + r0 * m, m, (int)b, m, m);
  cp_async_wait_all();
  __syncthreads();
  // phase 1: partials of this leaf; G = 8 consecutive lanes per (rank column, X
  // column) output split the rows (stride G), then a fixed butterfly over the group
  constexpr int G = 8;
  double* myp = P.part + L * (int64_t)kt * m;
  for (int base = 0; base < kt * m; base += blockDim.x / G) {
    const int o = base + (int)threadIdx.x / G, g = (int)threadIdx.x % G;
    double s = 0.0;
    if (o < kt * m) {
      const int a = o / m, c = o - a * m;
      for (int64_t r = g; r < b; r += G) s = fma(Vs[r * kt + a], Xs[r * m + c], s);
    }
#pragma unroll
    for (int w = 1; w < G; w <<= 1) s += __shfl_xor_sync(0xffffffffu, s, w);
    if (o < kt * m && g == 0) myp[o] = s;
  }
  cooperative_groups::this_grid().sync();  // every leaf's partials written
  // phase 2a: t of the sibling nodes, thread per (level, rank column, X column)
  for (int l = 1; l <= p; ++l) {
    const int k = P.k[l - 1];
    const int64_t span = (int64_t)1 << (p - l);
    const int64_t first = ((L >> (p - l)) ^ 1) * span;  // first leaf of the sibling node
    for (int o = threadIdx.x; o < k * m; o += blockDim.x) {
      const int64_t e = P.koff[l - 1] * m + o;
      double s = 0.0;
      int64_t L2 = first;
      for (; L2 + 4 <= first + span; L2 += 4) {  // 4 independent loads in flight, summed in order
        const double v0 = ldg_cg(P.part + L2 * kt * m + e), v1 = ldg_cg(P.part + (L2 + 1) * kt * m + e);
        const double v2 = ldg_cg(P.part + (L2 + 2) * kt * m + e), v3 = ldg_cg(P.part + (L2 + 3) * kt * m + e);
        s += v0; s += v1; s += v2; s += v3;
      }
      for (; L2 < first + span; ++L2) s += ldg_cg(P.part + L2 * kt * m + e);
      Ts[e] = s;
    }
  }
  __syncthreads();
  // phase 2b: Y(I_L) = D_L X(I_L) + U(I_L) T; G consecutive lanes per output
  // split the extended row, fixed butterfly over the group
  for (int64_t base = 0; base < b * m; base += blockDim.x / G) {
    const int64_t o = base + (int)threadIdx.x / G;
    const int g = (int)threadIdx.x % G;
    double s = 0.0;
    if (o < b * m) {
      const int64_t r = o / m;
      const int c = (int)(o - r * m);
      for (int64_t j = g; j < b; j += G) s = fma(Ds[r * zd + j], Xs[j * m + c], s);
      for (int a = g; a < kt; a += G) s = fma(Us[r * kt + a], Ts[a * m + c], s);
    }
#pragma unroll
    for (int w = 1; w < G; w <<= 1) s += __shfl_xor_sync(0xffffffffu, s, w);
    if (o < b * m && g == 0) P.Y[(r0 + (o / m)) * m + (o % m)] = s;
  }
}

}  // namespace hm
