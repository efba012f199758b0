// hm_tree.cuh — HSS tree levels, nrhs >= 2, DMMA fragments.
//
// Upsweep (Fig. 5 right):   x_l[i] = W_{l,i}^T [x_{l+1}[2i]; x_{l+1}[2i+1]]
// Coupling + downsweep (reading G1), one level at a time:
//                                      y_l[2q+w] = R_{l-1,q}[w] y_{l-1}[q] + S_w x_l[2q+1-w]
// One CTA (8 warps) owns a PAIR of nodes: the coefficient blocks it needs
// (the four children of an up pair; the sibling pair's x and the parent's y of
// a down pair) are staged once in shared memory with a padded row stride, so
// every warp reads its DMMA B fragments from shared memory; generators (W, R,
// B) stream from HBM as 128-bit A fragments. Big levels run as one launch per
// level; the small top levels run in ONE persistent cooperative launch with a
// grid-wide barrier between levels (hss_tree_sweep_kernel).
#pragma once
#include <cooperative_groups.h>

#include "hm_fast.cuh"

namespace hm {

struct TreeParams {
  const double* W;       // [2^p-2][2k][k]
  const double* R;       // [2^p-2][2k][k]
  const double* B;       // [2^p-1][2][k][k]
  double* xh;            // level-major coefficient blocks [k][m]
  double* yh;
  const double* R_root;  // optional (distributed subtree): translation of the subtree root,
  const double* y_root;  //   [2k][k], and its y block [k][m]: adds R_root[w] y_root at level 1
  int32_t m;
  int32_t bt;            // 1: adjoint cores S'_0 = B21^T, S'_1 = B12^T
};

// Staged blocks hold mpad = ceil(m / 8NT) * 8NT columns (zero padded) so every
// column chunk reads inside its row. Row strides (in doubles) for conflict-free
// 64-bit fragment loads — a warp's 64-bit shared load is served per half-warp
// (16 lanes: i = lane>>2 in 0..3, j = lane&3), conflict-free iff the 16
// addresses fall in 16 distinct 8-byte bank pairs (d mod 16 distinct):
//   transposed B fragments read rows r + j, d = j zs + i: zs = 4 (mod 8);
//   row-major B fragments read rows r + 2j, d = 2 j zs + i: zs = 2 (mod 4).
// (Measured with ncu: strides 8 (mod 16) / 4 (mod 8) gave 2-way conflicts on
// every load, l1tex__data_bank_conflicts = 1/2 of the wavefronts.)
#ifndef HM_TREE_UP_HQ
#define HM_TREE_UP_HQ 4  // k-steps of W per register chunk in the up kernel (measured, r01_tuning.md)
#endif
__host__ __device__ constexpr int tree_mpad(int m, int nt) { return (m + nt * 8 - 1) / (nt * 8) * (nt * 8); }
__host__ __device__ constexpr int tree_up_stride(int mpad) { return mpad + 4; }
__host__ __device__ constexpr int tree_down_stride(int mpad) { return mpad + 2; }
__host__ __device__ constexpr int64_t tree_smem_doubles(int kt, int m, int nt) {
  return (4ll * kt * tree_up_stride(tree_mpad(m, nt)) > 3ll * kt * tree_down_stride(tree_mpad(m, nt)))
             ? 4ll * kt * tree_up_stride(tree_mpad(m, nt))
             : 3ll * kt * tree_down_stride(tree_mpad(m, nt));
}

// Up: CTA task for the node pair (2r, 2r+1) of level l (children: 4 consecutive
// level-(l+1) blocks). 4 warps per node: rank-column group mg = w % MG, column
// chunks ck = w / MG, w / MG + 4/MG, ...
template <int KT, int NT, bool COH>
__device__ __forceinline__ void tree_up_pair(const TreeParams& P, int l, int64_t r, double* sm) {
  constexpr int MG = KT / 16;
  constexpr int CKS = 4 / MG;  // chunk step per node
  constexpr int NQ = KT / 2;   // k-steps of the 2k-row contraction
  const int m = P.m;
  const int mp = tree_mpad(m, NT);
  const int zs = tree_up_stride(mp);
  const int64_t km = (int64_t)KT * m;
  const int64_t n0 = 2 * r;  // level l >= 1 has an even number of nodes
  const int nodes = 2;
  stage_rows_async(sm, zs, P.xh + ((1ll << (l + 1)) - 2 + 2 * n0) * km, m, 2 * nodes * KT, m, mp);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nd = w >> 2, sub = w & 3;
  const int i = lane >> 2, j = lane & 3;
  const int64_t node = n0 + nd;
  const int mg = sub % MG;
  // The warp's slice of W (2k rows x 16 rank columns, one LDG.128 per k-step)
  // streams in chunks of HQ k-steps; the first chunk is requested before the
  // staged children are waited for, so the generator stream and the staging
  // overlap. HQ < NQ bounds the registers (more CTAs per SM).
  constexpr int HQ = HM_TREE_UP_HQ < NQ ? HM_TREE_UP_HQ : NQ;
  const double* ap = P.W + ((1ll << l) - 2 + node) * 2 * KT * KT + mg * 16 + (int64_t)j * KT + 2 * i;
  double2 a[HQ];
#pragma unroll
  for (int q = 0; q < HQ; ++q) a[q] = ldg_stream2(ap + (int64_t)q * 4 * KT);
  cp_async_wait_all();
  __syncthreads();
  // the 4 warps of a node split MG rank groups x column chunks; narrower chunks
  // (NTU = NT * MG / 4) keep all 4 busy when MG < 4 (k = 16, 32)
  constexpr int NTU = (NT * MG / 4) >= 1 ? (NT * MG / 4) : 1;
  {
    const double* bp = sm + nd * 2 * KT * zs + j * zs + i;
    double* out = P.xh + ((1ll << l) - 2 + node) * km + (int64_t)mg * 16 * m;
    const int nck = mp / (NTU * 8);
    bool loaded = true;  // a[] holds chunk 0
    for (int ck = sub / MG; ck < nck; ck += CKS) {
      const int c0 = ck * NTU * 8;
      double acc[2][NTU][2];
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int nt = 0; nt < NTU; ++nt) acc[t][nt][0] = acc[t][nt][1] = 0.0;
#pragma unroll
      for (int q0 = 0; q0 < NQ; q0 += HQ) {
        if (!loaded) {
#pragma unroll
          for (int q = 0; q < HQ; ++q) a[q] = ldg_stream2(ap + (int64_t)(q0 + q) * 4 * KT);
        }
        loaded = false;
#pragma unroll
        for (int q = 0; q < HQ; ++q) {
          double bf[NTU];
#pragma unroll
          for (int nt = 0; nt < NTU; ++nt) bf[nt] = bp[(q0 + q) * 4 * zs + c0 + nt * 8];
#pragma unroll
          for (int nt = 0; nt < NTU; ++nt) dmma(acc[0][nt][0], acc[0][nt][1], a[q].x, bf[nt]);
#pragma unroll
          for (int nt = 0; nt < NTU; ++nt) dmma(acc[1][nt][0], acc[1][nt][1], a[q].y, bf[nt]);
        }
      }
      store_transposed<1, NTU>(acc, out, m, c0, m, lane);
    }
  }
  __syncthreads();  // shared memory is reused by the next task
}

// Down: CTA task for the sibling pair (2q, 2q+1) of level l: stage x_l[2q],
// x_l[2q+1] (contiguous) and y_{l-1}[q]; warp (nd, sub) computes rows of
// y_l[2q+nd] = R_{l-1,q}[nd] y_{l-1}[q] + S_nd x_l[2q+1-nd].
template <int KT, int NT, bool COH>
__device__ __forceinline__ void tree_down_pair(const TreeParams& P, int l, int64_t q, double* sm) {
  constexpr int RGS = KT / 8;
  const int m = P.m;
  const int mp = tree_mpad(m, NT);
  const int zs = tree_down_stride(mp);
  const int64_t km = (int64_t)KT * m;
  stage_rows_async(sm, zs, P.xh + ((1ll << l) - 2 + 2 * q) * km, m, 2 * KT, m, mp);
  const bool root_term = (l == 1 && P.R_root != nullptr);
  if (l >= 2) stage_rows_async(sm + 2 * KT * zs, zs, P.yh + ((1ll << (l - 1)) - 2 + q) * km, m, KT, m, mp);
  if (root_term) stage_rows_async(sm + 2 * KT * zs, zs, P.y_root, m, KT, m, mp);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nd = w >> 2, sub = w & 3;
  const int64_t j = 2 * q + nd;
  // A: S = B12 (nd 0) / B21 (nd 1); adjoint (bt): S' = (the other core)^T
  const double* S = P.B + (((1ll << (l - 1)) - 1 + q) * 2 + (P.bt ? 1 - nd : nd)) * KT * KT;
  const double* Rw = (l >= 2) ? P.R + (((1ll << (l - 1)) - 2 + q) * 2 * KT + nd * KT) * KT
                     : (root_term ? P.R_root + (int64_t)nd * KT * KT : nullptr);
  const double* Zx = sm + (1 - nd) * KT * zs;  // the sibling's x
  const double* Zy = sm + 2 * KT * zs;
  double* yo = P.yh + ((1ll << l) - 2 + j) * km;
  const int nck = mp / (NT * 8);
  const int ntask = RGS * nck;
  const int i = lane >> 2, jj = lane & 3;
  // every A fragment of both terms of a task is requested before the first
  // DMMA — for the first task before the staged blocks are waited for
  constexpr int NQ = KT / 8;
  double2 aR[NQ][1], aS[NQ][1];
  auto load_task = [&](int t) {
    const int rg = t % RGS;
    const double* bR = Rw ? Rw + (int64_t)(rg * 8 + i) * KT + 2 * jj : nullptr;
    const double* bS = P.bt ? S + (int64_t)(2 * jj) * KT + rg * 8 + i : S + (int64_t)(rg * 8 + i) * KT + 2 * jj;
#pragma unroll
    for (int q2 = 0; q2 < NQ; ++q2) {
      aR[q2][0] = bR ? ldg_stream2(bR + 8 * q2) : make_double2(0.0, 0.0);
      // S'[row][k] = S[k][row]: the two k-indices 8 q2 + 2 jj (+1) are rows of S
      aS[q2][0] = P.bt ? make_double2(ldg_stream(bS + (int64_t)8 * q2 * KT), ldg_stream(bS + (int64_t)(8 * q2 + 1) * KT))
                       : ldg_stream2(bS + 8 * q2);
    }
  };
  if (sub < ntask) load_task(sub);
  cp_async_wait_all();
  __syncthreads();
  for (int t = sub; t < ntask; t += 4) {
    const int rg = t % RGS, ck = t / RGS;
    const int c0 = ck * NT * 8;
    double acc[1][NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[0][nt][0] = acc[0][nt][1] = 0.0;
    bool colok[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) colok[nt] = true;
    if (Rw) rm_group<1, NT, false, false, NQ>(acc, aR, Zy + c0, zs, 0, NQ, colok, lane);
    rm_group<1, NT, false, false, NQ>(acc, aS, Zx + c0, zs, 0, NQ, colok, lane);
    if (t + 4 < ntask) load_task(t + 4);
    double* y = yo + (int64_t)(8 * rg + i) * m;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int c = c0 + nt * 8 + 2 * jj;
      if (c + 1 < m) {
        y[c] = acc[0][nt][0];
        y[c + 1] = acc[0][nt][1];
      } else if (c < m) {
        y[c] = acc[0][nt][0];
      }
    }
  }
  __syncthreads();
}

template <int KT, int NT, int MINB>
__global__ void __launch_bounds__(256, MINB) hss_up_pair_kernel(const TreeParams P, int l) {
  extern __shared__ double sm[];
  tree_up_pair<KT, NT, false>(P, l, blockIdx.x, sm);
}

template <int KT, int NT, int MINB>
__global__ void __launch_bounds__(256, MINB) hss_down_pair_kernel(const TreeParams P, int l) {
  extern __shared__ double sm[];
  tree_down_pair<KT, NT, false>(P, l, blockIdx.x, sm);
}

// A fragments of one down task (row group rg of y = Rw y_parent + S x_sib), as in
// tree_down_pair's load_task.
template <int KT>
__device__ __forceinline__ void down_load_task(double2 (&aR)[KT / 8][1], double2 (&aS)[KT / 8][1], const double* S,
                                               const double* Rw, int bt, int rg, int lane) {
  const int i = lane >> 2, jj = lane & 3;
  const double* bR = Rw + (int64_t)(rg * 8 + i) * KT + 2 * jj;
  const double* bS = bt ? S + (int64_t)(2 * jj) * KT + rg * 8 + i : S + (int64_t)(rg * 8 + i) * KT + 2 * jj;
#pragma unroll
  for (int q2 = 0; q2 < KT / 8; ++q2) {
    aR[q2][0] = ldg_stream2(bR + 8 * q2);
    aS[q2][0] = bt ? make_double2(ldg_stream(bS + (int64_t)8 * q2 * KT), ldg_stream(bS + (int64_t)(8 * q2 + 1) * KT))
                   : ldg_stream2(bS + 8 * q2);
  }
}
// One down task: rows 8 rg .. 8 rg + 7, columns c0 .. c0 + 8 NT - 1 of
// y = Rw y_parent + S x_sib from the staged blocks Zy, Zx (row stride zs), into
// registers (down_task_acc), then stored to yo (row stride ldo, columns < lim).
template <int KT, int NT>
__device__ __forceinline__ void down_task_acc(double (&acc)[1][NT][2], const double2 (&aR)[KT / 8][1],
                                              const double2 (&aS)[KT / 8][1], const double* Zx, const double* Zy,
                                              int zs, int c0, int lane) {
  constexpr int NQ = KT / 8;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) acc[0][nt][0] = acc[0][nt][1] = 0.0;
  bool colok[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) colok[nt] = true;
  rm_group<1, NT, false, false, NQ>(acc, aR, Zy + c0, zs, 0, NQ, colok, lane);
  rm_group<1, NT, false, false, NQ>(acc, aS, Zx + c0, zs, 0, NQ, colok, lane);
}
template <int NT>
__device__ __forceinline__ void down_store(const double (&acc)[1][NT][2], double* yo, int64_t ldo, int lim, int rg,
                                           int c0, int lane) {
  const int i = lane >> 2, jj = lane & 3;
  double* y = yo + (int64_t)(8 * rg + i) * ldo;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int c = c0 + nt * 8 + 2 * jj;
    if (c + 1 < lim) {
      y[c] = acc[0][nt][0];
      y[c + 1] = acc[0][nt][1];
    } else if (c < lim) {
      y[c] = acc[0][nt][0];
    }
  }
}
template <int KT, int NT>
__device__ __forceinline__ void down_task(const double2 (&aR)[KT / 8][1], const double2 (&aS)[KT / 8][1],
                                          const double* Zx, const double* Zy, int zs, double* yo, int64_t ldo, int lim,
                                          int rg, int c0, int lane) {
  double acc[1][NT][2];
  down_task_acc<KT, NT>(acc, aR, aS, Zx, Zy, zs, c0, lane);
  down_store<NT>(acc, yo, ldo, lim, rg, c0, lane);
}

// Two downsweep levels in one launch (l >= 2): CTA = the level-(l-1) node q.
// Stages x_l[2q..2q+1], y_{l-1}[q] and the four grandchildren x_{l+1}[4q..4q+3]
// at once; phase A (4 warps per node) forms y_l[2q + nd] = R_{l-1,q}[nd] y_{l-1}[q]
// + S_nd x_l[2q+1-nd] in shared memory only; phase B (2 warps per node) forms
// y_{l+1}[4q + c] from it and writes them. y_l never goes to HBM: one write +
// one re-read of the level's blocks saved. Config 4, down levels 11..14 at
// nrhs 8 / 16: 119 / 176 -> 103 / 135 us; 11..15 at nrhs 32 (ALIAS layout,
// 3 CTAs per SM): 470 -> 420-430 us. (The 9-block layout at 32 columns, 78 KB
// per CTA and 2 CTAs per SM, took 345 us for levels 14 + 15 against 108 + 209 us
// as two pair launches; 16-column windows that re-read the generators 484 us.)
__host__ __device__ constexpr int64_t tree_down_two_doubles(int kt, int m, int nt, bool alias = false) {
  return (alias ? 7ll : 9ll) * kt * tree_down_stride(tree_mpad(m, nt));
}
// ALIAS (every warp has at most one phase-A task): y_l is written over the
// staged x_l pair after a barrier — 7 blocks instead of 9, so 3 CTAs per SM fit
// at k = 32 with 32 columns. The grandchildren's x_{l+1} are a second cp.async
// group, still landing while phase A computes.
template <int KT, int NT, int MINB, bool ALIAS>
__global__ void __launch_bounds__(256, MINB) hss_down_two_kernel(const TreeParams P, int l) {
  extern __shared__ double sm[];
  constexpr int RGS = KT / 8, NQ = KT / 8;
  const int m = P.m, mp = tree_mpad(m, NT), zs = tree_down_stride(mp);
  const int64_t km = (int64_t)KT * m;
  const int64_t q = blockIdx.x;
  const int blk = KT * zs;
  double* Xl = sm;                                // x_l[2q], x_l[2q+1]
  double* Yp = sm + 2 * blk;                      // y_{l-1}[q]
  double* Yl = ALIAS ? sm : sm + 3 * blk;         // y_l[2q], y_l[2q+1]
  double* Xc = sm + (ALIAS ? 3 : 5) * blk;        // x_{l+1}[4q .. 4q+3]
  stage_rows_async(Xl, zs, P.xh + ((1ll << l) - 2 + 2 * q) * km, m, 2 * KT, m, mp);
  stage_rows_async(Yp, zs, P.yh + ((1ll << (l - 1)) - 2 + q) * km, m, KT, m, mp);
  cp_async_commit_group();
  stage_rows_async(Xc, zs, P.xh + ((1ll << (l + 1)) - 2 + 4 * q) * km, m, 4 * KT, m, mp);
  cp_async_commit_group();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nck = mp / (NT * 8), ntask = RGS * nck;
  double2 aR[NQ][1], aS[NQ][1];
  {  // phase A: level l
    const int nd = w >> 2, sub = w & 3;
    const double* S = P.B + (((1ll << (l - 1)) - 1 + q) * 2 + (P.bt ? 1 - nd : nd)) * KT * KT;
    const double* Rw = P.R + (((1ll << (l - 1)) - 2 + q) * 2 * KT + nd * KT) * KT;
    if (sub < ntask) down_load_task<KT>(aR, aS, S, Rw, P.bt, sub % RGS, lane);
    cp_async_wait_groups<1>();  // x_l, y_{l-1} landed (this thread's copies) ...
    __syncthreads();            // ... and everyone's
    if constexpr (ALIAS) {
      double acc[1][NT][2];
      const bool has = sub < ntask;
      if (has) down_task_acc<KT, NT>(acc, aR, aS, Xl + (1 - nd) * blk, Yp, zs, (sub / RGS) * NT * 8, lane);
      __syncthreads();  // every read of x_l / y_{l-1} done: y_l overwrites x_l
      if (has) down_store<NT>(acc, Yl + nd * blk, zs, mp, sub % RGS, (sub / RGS) * NT * 8, lane);
    } else {
      for (int t = sub; t < ntask; t += 4) {
        down_task<KT, NT>(aR, aS, Xl + (1 - nd) * blk, Yp, zs, Yl + nd * blk, zs, mp, t % RGS, (t / RGS) * NT * 8,
                          lane);
        if (t + 4 < ntask) down_load_task<KT>(aR, aS, S, Rw, P.bt, (t + 4) % RGS, lane);
      }
    }
  }
  cp_async_wait_groups<0>();  // x_{l+1} landed
  {  // phase B: level l + 1, node 4q + nd4 under the level-l node 2q + pp
    const int nd4 = w >> 1, sub = w & 1, pp = nd4 >> 1, nd = nd4 & 1;
    const int64_t qq = 2 * q + pp;
    const double* S = P.B + (((1ll << l) - 1 + qq) * 2 + (P.bt ? 1 - nd : nd)) * KT * KT;
    const double* Rw = P.R + (((1ll << l) - 2 + qq) * 2 * KT + nd * KT) * KT;
    if (sub < ntask) down_load_task<KT>(aR, aS, S, Rw, P.bt, sub % RGS, lane);
    __syncthreads();  // y_l complete
    double* yo = P.yh + ((1ll << (l + 1)) - 2 + 4 * q + nd4) * km;
    for (int t = sub; t < ntask; t += 2) {
      down_task<KT, NT>(aR, aS, Xc + (nd4 ^ 1) * blk, Yl + pp * blk, zs, yo, m, m, t % RGS, (t / RGS) * NT * 8, lane);
      if (t + 2 < ntask) down_load_task<KT>(aR, aS, S, Rw, P.bt, (t + 2) % RGS, lane);
    }
  }
}

// Levels [lo, hi] of both sweeps in one cooperative launch: up l = hi-1 .. lo
// (reading x_{l+1}), then down l = lo' .. hi where lo' = lo for the down pass
// (down starts at level 1 when lo == 1). Grid barrier between levels.
template <int KT, int NT>
__global__ void __launch_bounds__(256) hss_tree_sweep_kernel(const TreeParams P, int up_from, int up_to, int down_from,
                                                              int down_to) {
  namespace cg = cooperative_groups;
  extern __shared__ double sm[];
  cg::grid_group grid = cg::this_grid();
  bool first = true;
  for (int l = up_from; l >= up_to; --l) {
    if (!first) grid.sync();
    first = false;
    const int64_t pairs = ((1ll << l) + 1) / 2;
    for (int64_t r = blockIdx.x; r < pairs; r += gridDim.x) tree_up_pair<KT, NT, true>(P, l, r, sm);
  }
  for (int l = down_from; l <= down_to; ++l) {
    if (!first) grid.sync();
    first = false;
    const int64_t pairs = 1ll << (l - 1);
    for (int64_t q = blockIdx.x; q < pairs; q += gridDim.x) tree_down_pair<KT, NT, true>(P, l, q, sm);
  }
}

// ------------------------------------------ big levels, generators staged --
// The same pair tasks as tree_up_pair / tree_down_pair for the big levels (one
// launch per level), with the node pair's generators (W; or R and the cores)
// staged in shared memory together with the coefficient blocks: every byte a
// CTA needs is requested at once (one cp.async wait), and the A fragments come
// from shared memory. Strides: W rows KT + 4 (LDS.128 of rows 4q + j, columns
// 2i: conflict-free), R / core rows KT + 8 (rows 8 rg + i, columns 8 q + 2 j).
__host__ __device__ constexpr int tree_ws(int kt) { return kt + 4; }
__host__ __device__ constexpr int tree_rs(int kt) { return kt + 8; }
__host__ __device__ constexpr int64_t tree_up_stage_doubles(int kt, int m, int nt) {
  return 4ll * kt * tree_up_stride(tree_mpad(m, nt)) + 4ll * kt * tree_ws(kt);
}
__host__ __device__ constexpr int64_t tree_down_stage_doubles(int kt, int m, int nt) {
  return 3ll * kt * tree_down_stride(tree_mpad(m, nt)) + 4ll * kt * tree_rs(kt);
}

template <int KT, int NT>
__global__ void __launch_bounds__(256) hss_up_stage_kernel(const TreeParams P, int l) {
  extern __shared__ double sm[];
  constexpr int MG = KT / 16, CKS = 4 / MG, NQ = KT / 2, WS = tree_ws(KT);
  const int m = P.m, mp = tree_mpad(m, NT), zs = tree_up_stride(mp);
  const int64_t km = (int64_t)KT * m, n0 = 2 * (int64_t)blockIdx.x;
  double* Zc = sm;                 // the 4 children blocks
  double* Ws = sm + 4 * KT * zs;   // W of the 2 nodes, [2][2KT][WS]
  stage_rows_async(Zc, zs, P.xh + ((1ll << (l + 1)) - 2 + 2 * n0) * km, m, 4 * KT, m, mp);
  stage_rows_async(Ws, WS, P.W + ((1ll << l) - 2 + n0) * 2 * KT * KT, KT, 4 * KT, KT, KT);
  cp_async_wait_all();
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nd = w >> 2, sub = w & 3, mg = sub % MG;
  const int i = lane >> 2, j = lane & 3;
  constexpr int NTU = (NT * MG / 4) >= 1 ? (NT * MG / 4) : 1;
  const double* ap = Ws + (nd * 2 * KT + j) * WS + mg * 16 + 2 * i;
  const double* bp = Zc + nd * 2 * KT * zs + j * zs + i;
  double* out = P.xh + ((1ll << l) - 2 + n0 + nd) * km + (int64_t)mg * 16 * m;
  const int nck = mp / (NTU * 8);
  for (int ck = sub / MG; ck < nck; ck += CKS) {
    const int c0 = ck * NTU * 8;
    double acc[2][NTU][2];
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int nt = 0; nt < NTU; ++nt) acc[t][nt][0] = acc[t][nt][1] = 0.0;
#pragma unroll 4
    for (int q = 0; q < NQ; ++q) {
      const double2 a = *reinterpret_cast<const double2*>(ap + q * 4 * WS);
#pragma unroll
      for (int nt = 0; nt < NTU; ++nt) {
        const double bf = bp[q * 4 * zs + c0 + nt * 8];
        dmma(acc[0][nt][0], acc[0][nt][1], a.x, bf);
        dmma(acc[1][nt][0], acc[1][nt][1], a.y, bf);
      }
    }
    store_transposed<1, NTU>(acc, out, m, c0, m, lane);
  }
}

template <int KT, int NT>
__global__ void __launch_bounds__(256) hss_down_stage_kernel(const TreeParams P, int l) {
  extern __shared__ double sm[];
  constexpr int RGS = KT / 8, NQ = KT / 8, RS = tree_rs(KT);
  const int m = P.m, mp = tree_mpad(m, NT), zs = tree_down_stride(mp);
  const int64_t km = (int64_t)KT * m, q = blockIdx.x;
  double* Zx = sm;                       // x of the sibling pair
  double* Zy = sm + 2 * KT * zs;         // y of the parent
  double* Sb = sm + 3 * KT * zs;         // the two cores [2][KT][RS]
  double* Rb = Sb + 2 * KT * RS;         // the parent's R [2KT][RS]
  const bool has_r = l >= 2 || P.R_root != nullptr;
  stage_rows_async(Zx, zs, P.xh + ((1ll << l) - 2 + 2 * q) * km, m, 2 * KT, m, mp);
  if (l >= 2) stage_rows_async(Zy, zs, P.yh + ((1ll << (l - 1)) - 2 + q) * km, m, KT, m, mp);
  else if (P.R_root) stage_rows_async(Zy, zs, P.y_root, m, KT, m, mp);
  stage_rows_async(Sb, RS, P.B + ((1ll << (l - 1)) - 1 + q) * 2 * KT * KT, KT, 2 * KT, KT, KT);
  if (has_r)
    stage_rows_async(Rb, RS, l >= 2 ? P.R + ((1ll << (l - 1)) - 2 + q) * 2 * KT * KT : P.R_root, KT, 2 * KT, KT, KT);
  cp_async_wait_all();
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nd = w >> 2, sub = w & 3;
  const int i = lane >> 2, jj = lane & 3;
  const double* S = Sb + (P.bt ? 1 - nd : nd) * KT * RS;
  const double* Rw = Rb + nd * KT * RS;
  const double* Zs = Zx + (1 - nd) * KT * zs;  // the sibling's x
  double* yo = P.yh + ((1ll << l) - 2 + 2 * q + nd) * km;
  const int nck = mp / (NT * 8);
  bool colok[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) colok[nt] = true;
  for (int t = sub; t < RGS * nck; t += 4) {
    const int rg = t % RGS, ck = t / RGS, c0 = ck * NT * 8;
    double2 aR[NQ][1], aS[NQ][1];
#pragma unroll
    for (int q2 = 0; q2 < NQ; ++q2) {
      aR[q2][0] = has_r ? *reinterpret_cast<const double2*>(Rw + (rg * 8 + i) * RS + 8 * q2 + 2 * jj)
                        : make_double2(0.0, 0.0);
      // adjoint: S'[row][k] = S[k][row]
      aS[q2][0] = P.bt ? make_double2(S[(8 * q2 + 2 * jj) * RS + rg * 8 + i], S[(8 * q2 + 2 * jj + 1) * RS + rg * 8 + i])
                       : *reinterpret_cast<const double2*>(S + (rg * 8 + i) * RS + 8 * q2 + 2 * jj);
    }
    double acc[1][NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[0][nt][0] = acc[0][nt][1] = 0.0;
    if (has_r) rm_group<1, NT, false, false, NQ>(acc, aR, Zy + c0, zs, 0, NQ, colok, lane);
    rm_group<1, NT, false, false, NQ>(acc, aS, Zs + c0, zs, 0, NQ, colok, lane);
    double* y = yo + (int64_t)(8 * rg + i) * m;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int c = c0 + nt * 8 + 2 * jj;
      if (c + 1 < m) {
        y[c] = acc[0][nt][0];
        y[c + 1] = acc[0][nt][1];
      } else if (c < m) {
        y[c] = acc[0][nt][0];
      }
    }
  }
}

// ------------------------------------------------ dataflow tree (one launch) --
// Every level of the upsweep and of the coupling / downsweep (Fig. 5 right,
// P:689-716) in ONE launch without grid barriers: CTAs draw pair tasks from a
// ticket counter in dependency order (up: level up_from .. 1, then down:
// level 1 .. down_last) and a task waits only for the flags of the tasks it
// reads — an up pair for its two child pairs, a down pair for its parent's pair
// and (x computed in this launch) the up pair of its own level. A task only
// waits for smaller tickets, which CTAs already running hold, so the schedule
// needs no co-residency. Levels overlap: a pair starts as soon as its inputs
// exist, not when the whole previous level is done, and the generators (W; R
// and the cores), which never wait, are requested before the flag wait.
//
// flags: [0] ticket, then up flags (pair (l, r) at 2^(l-1) - 1 + r), then down
// flags (offset 2^up_from, pair (l, q) at 2^(l-1) - 1 + q); zeroed before the
// launch. A flag is released (bar.sync, then st.release.gpu by thread 0) once the
// pair's blocks are stored; readers stage them with cp.async.cg / ld.cg (L2).
struct FlowParams {
  TreeParams T;
  unsigned* flags;
  int32_t up_from;    // upsweep levels up_from .. 1 (0: none)
  int32_t down_last;  // downsweep levels 1 .. down_last (0: none)
  unsigned long long* trace;  // HM_FLOW_TRACE builds: per task [start, waited, staged, done, signalled, smid]
};
#ifndef HM_FLOW_TRACE
#define HM_FLOW_TRACE 0
#endif
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// task trace (HM_FLOW_TRACE builds only): thread 0 stamps the task's phases
__device__ __forceinline__ void flow_stamp(unsigned long long* ft, int slot) {
  if (HM_FLOW_TRACE && ft && threadIdx.x == 0) ft[slot] = gtimer();
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// thread 0 waits for the flags, then the CTA proceeds (bar.sync orders the
// other threads' loads after thread 0's acquire)
#ifndef HM_FLOW_SPLIT
#define HM_FLOW_SPLIT 2  // independent partial sums per up-task accumulator
#endif
#ifndef HM_FLOW_SLEEP
#define HM_FLOW_SLEEP 32  // ns between polls of a flag (0: spin)
#endif
#ifndef HM_FLOW_FENCE
#define HM_FLOW_FENCE 0  // 1: __threadfence() before the release store (the release alone orders the CTA's stores after bar.sync)
#endif
__device__ __forceinline__ void flow_wait(const unsigned* f0, const unsigned* f1) {
  if (threadIdx.x == 0) {
    if (f0)
      while (ld_acquire_u32(f0) == 0)
        if (HM_FLOW_SLEEP) __nanosleep(HM_FLOW_SLEEP);
    if (f1)
      while (ld_acquire_u32(f1) == 0)
        if (HM_FLOW_SLEEP) __nanosleep(HM_FLOW_SLEEP);
  }
  __syncthreads();
}
__device__ __forceinline__ void flow_signal(unsigned* f) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (HM_FLOW_FENCE) __threadfence();
    st_release_u32(f, 1u);
  }
}

__host__ __device__ constexpr int64_t flow_smem_doubles(int kt, int m, int nt) {
  return tree_up_stage_doubles(kt, m, nt) > tree_smem_doubles(kt, m, nt) ? tree_up_stage_doubles(kt, m, nt)
                                                                         : tree_smem_doubles(kt, m, nt);
}

// Up pair (l, r) as hss_up_stage: W staged first, children after the wait.
template <int KT, int NT>
__device__ __forceinline__ void flow_up_pair(const TreeParams& P, int l, int64_t r, double* sm, const unsigned* f0,
                                             const unsigned* f1, unsigned long long* ft) {
  constexpr int MG = KT / 16, CKS = 4 / MG, NQ = KT / 2, WS = tree_ws(KT);
  const int m = P.m, mp = tree_mpad(m, NT), zs = tree_up_stride(mp);
  const int64_t km = (int64_t)KT * m, n0 = 2 * r;
  double* Zc = sm;
  double* Ws = sm + 4 * KT * zs;
  stage_rows_async(Ws, WS, P.W + ((1ll << l) - 2 + n0) * 2 * KT * KT, KT, 4 * KT, KT, KT);
  flow_wait(f0, f1);
  flow_stamp(ft, 1);
  stage_rows_async(Zc, zs, P.xh + ((1ll << (l + 1)) - 2 + 2 * n0) * km, m, 4 * KT, m, mp);
  cp_async_wait_all();
  __syncthreads();
  flow_stamp(ft, 2);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nd = w >> 2, sub = w & 3, mg = sub % MG;
  const int i = lane >> 2, j = lane & 3;
  constexpr int NTU = (NT * MG / 4) >= 1 ? (NT * MG / 4) : 1;
  const double* ap = Ws + (nd * 2 * KT + j) * WS + mg * 16 + 2 * i;
  const double* bp = Zc + nd * 2 * KT * zs + j * zs + i;
  double* out = P.xh + ((1ll << l) - 2 + n0 + nd) * km + (int64_t)mg * 16 * m;
  const int nck = mp / (NTU * 8);
  for (int ck = sub / MG; ck < nck; ck += CKS) {
    const int c0 = ck * NTU * 8;
    // HM_FLOW_SPLIT independent partial sums over the k-steps: the dependent
    // DMMA chain (the task's latency on the tree's critical path) is that much
    // shorter; the partials are added in a fixed order at the end
    double acc[HM_FLOW_SPLIT][2][NTU][2];
#pragma unroll
    for (int h = 0; h < HM_FLOW_SPLIT; ++h)
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int nt = 0; nt < NTU; ++nt) acc[h][t][nt][0] = acc[h][t][nt][1] = 0.0;
#pragma unroll 2
    for (int q0 = 0; q0 < NQ; q0 += HM_FLOW_SPLIT) {
#pragma unroll
      for (int h = 0; h < HM_FLOW_SPLIT; ++h) {
        const int q = q0 + h;
        const double2 a = *reinterpret_cast<const double2*>(ap + q * 4 * WS);
#pragma unroll
        for (int nt = 0; nt < NTU; ++nt) {
          const double bf = bp[q * 4 * zs + c0 + nt * 8];
          dmma(acc[h][0][nt][0], acc[h][0][nt][1], a.x, bf);
          dmma(acc[h][1][nt][0], acc[h][1][nt][1], a.y, bf);
        }
      }
    }
#pragma unroll
    for (int h = 1; h < HM_FLOW_SPLIT; ++h)
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int nt = 0; nt < NTU; ++nt) {
          acc[0][t][nt][0] += acc[h][t][nt][0];
          acc[0][t][nt][1] += acc[h][t][nt][1];
        }
    store_transposed<1, NTU>(acc[0], out, m, c0, m, lane);
  }
}

// Down pair (l, q) as tree_down_pair: the first task's R / core fragments are
// requested before the wait, the coefficient blocks staged after it.
template <int KT, int NT>
__device__ __forceinline__ void flow_down_pair(const TreeParams& P, int l, int64_t q, double* sm, const unsigned* f0,
                                               const unsigned* f1, unsigned long long* ft) {
  constexpr int RGS = KT / 8;
  const int m = P.m;
  const int mp = tree_mpad(m, NT);
  const int zs = tree_down_stride(mp);
  const int64_t km = (int64_t)KT * m;
  const bool root_term = (l == 1 && P.R_root != nullptr);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nd = w >> 2, sub = w & 3;
  const int64_t j = 2 * q + nd;
  const double* S = P.B + (((1ll << (l - 1)) - 1 + q) * 2 + (P.bt ? 1 - nd : nd)) * KT * KT;
  const double* Rw = (l >= 2) ? P.R + (((1ll << (l - 1)) - 2 + q) * 2 * KT + nd * KT) * KT
                     : (root_term ? P.R_root + (int64_t)nd * KT * KT : nullptr);
  const double* Zx = sm + (1 - nd) * KT * zs;
  const double* Zy = sm + 2 * KT * zs;
  double* yo = P.yh + ((1ll << l) - 2 + j) * km;
  const int nck = mp / (NT * 8);
  const int ntask = RGS * nck;
  const int i = lane >> 2, jj = lane & 3;
  constexpr int NQ = KT / 8;
  double2 aR[NQ][1], aS[NQ][1];
  auto load_task = [&](int t) {
    const int rg = t % RGS;
    const double* bR = Rw ? Rw + (int64_t)(rg * 8 + i) * KT + 2 * jj : nullptr;
    const double* bS = P.bt ? S + (int64_t)(2 * jj) * KT + rg * 8 + i : S + (int64_t)(rg * 8 + i) * KT + 2 * jj;
#pragma unroll
    for (int q2 = 0; q2 < NQ; ++q2) {
      aR[q2][0] = bR ? ldg_stream2(bR + 8 * q2) : make_double2(0.0, 0.0);
      aS[q2][0] = P.bt ? make_double2(ldg_stream(bS + (int64_t)8 * q2 * KT), ldg_stream(bS + (int64_t)(8 * q2 + 1) * KT))
                       : ldg_stream2(bS + 8 * q2);
    }
  };
  if (sub < ntask) load_task(sub);
  flow_wait(f0, f1);
  flow_stamp(ft, 1);
  stage_rows_async(sm, zs, P.xh + ((1ll << l) - 2 + 2 * q) * km, m, 2 * KT, m, mp);
  if (l >= 2) stage_rows_async(sm + 2 * KT * zs, zs, P.yh + ((1ll << (l - 1)) - 2 + q) * km, m, KT, m, mp);
  if (root_term) stage_rows_async(sm + 2 * KT * zs, zs, P.y_root, m, KT, m, mp);
  cp_async_wait_all();
  __syncthreads();
  flow_stamp(ft, 2);
  for (int t = sub; t < ntask; t += 4) {
    const int rg = t % RGS, ck = t / RGS;
    const int c0 = ck * NT * 8;
    // the R and core terms in separate accumulators (two dependent DMMA chains
    // of half the length, summed at the end)
    double acc[1][NT][2], acs[1][NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[0][nt][0] = acc[0][nt][1] = acs[0][nt][0] = acs[0][nt][1] = 0.0;
    bool colok[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) colok[nt] = true;
    if (Rw) rm_group<1, NT, false, false, NQ>(acc, aR, Zy + c0, zs, 0, NQ, colok, lane);
    rm_group<1, NT, false, false, NQ>(acs, aS, Zx + c0, zs, 0, NQ, colok, lane);
    if (t + 4 < ntask) load_task(t + 4);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      acc[0][nt][0] += acs[0][nt][0];
      acc[0][nt][1] += acs[0][nt][1];
    }
    double* y = yo + (int64_t)(8 * rg + i) * m;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int c = c0 + nt * 8 + 2 * jj;
      if (c + 1 < m) {
        y[c] = acc[0][nt][0];
        y[c + 1] = acc[0][nt][1];
      } else if (c < m) {
        y[c] = acc[0][nt][0];
      }
    }
  }
}

template <int KT, int NT>
__global__ void __launch_bounds__(256, KT >= 64 ? 1 : 2) hss_tree_flow_kernel(const FlowParams F) {
  extern __shared__ double sm[];
  __shared__ unsigned s_ticket;
  const int L = F.up_from, DL = F.down_last;
  const unsigned n_up = L >= 1 ? (1u << L) - 1 : 0u;
  const unsigned n_all = n_up + (DL >= 1 ? (1u << DL) - 1 : 0u);
  unsigned* upf = F.flags + 1;
  unsigned* dnf = upf + (1u << L);
  if (threadIdx.x == 0) s_ticket = atomicAdd(F.flags, 1u);
  __syncthreads();
  unsigned t = s_ticket;
  while (t < n_all) {
    // the next ticket is drawn while this task runs (read after its last barrier)
    unsigned nxt = 0;
    if (threadIdx.x == 0) nxt = atomicAdd(F.flags, 1u);
    unsigned long long* ft = HM_FLOW_TRACE && F.trace ? F.trace + 6ull * t : nullptr;
    flow_stamp(ft, 0);
    if (HM_FLOW_TRACE && ft && threadIdx.x == 0) {
      unsigned smid;
      asm("mov.u32 %0, %smid;" : "=r"(smid));
      ft[5] = smid;
    }
    if (t < n_up) {
      const unsigned v = (1u << L) - t;  // in (2^(l-1), 2^l]
      const int l = 32 - __clz(v - 1);
      const int64_t r = (int64_t)t - ((1ll << L) - (1ll << l));
      const bool wait = l + 1 <= L;  // children computed in this launch
      flow_up_pair<KT, NT>(F.T, l, r, sm, wait ? upf + (1u << l) - 1 + 2 * r : nullptr,
                           wait ? upf + (1u << l) - 1 + 2 * r + 1 : nullptr, ft);
      flow_stamp(ft, 3);
      flow_signal(upf + (1u << (l - 1)) - 1 + r);
    } else {
      const unsigned u = t - n_up;
      const int l = 32 - __clz(u + 1);
      const int64_t q = (int64_t)u + 1 - (1ll << (l - 1));
      const unsigned* fy = l >= 2 ? dnf + (1u << (l - 2)) - 1 + (q >> 1) : nullptr;
      const unsigned* fx = l <= L ? upf + (1u << (l - 1)) - 1 + q : nullptr;
      flow_down_pair<KT, NT>(F.T, l, q, sm, fy, fx, ft);
      flow_stamp(ft, 3);
      flow_signal(dnf + (1u << (l - 1)) - 1 + q);
    }
    flow_stamp(ft, 4);
    if (threadIdx.x == 0) s_ticket = nxt;
    __syncthreads();
    t = s_ticket;
    __syncthreads();  // s_ticket is rewritten at the end of the next task
  }
}

// ---------------------------------------------------- Step 1 + 3 up levels --
// HSS Step 1 fused with the first three upsweep levels (Fig. 5 right,
// P:684-694), nrhs <= 8 NT (one column chunk), k = KT in {16, 32}. CTA = the
// 8 leaves under node (p-3, c): warp w computes x_p[8c + w] = V_i^T X(I_i)
// (the vt_batched product), keeps it in shared memory and writes it out; then
// the CTA computes the 4 level-(p-1) nodes, the 2 level-(p-2) nodes and the
// level-(p-3) node from shared memory (W^T [x_left; x_right], W streamed as
// 128-bit A fragments), writing every x block once (the downsweep's coupling
// reads them) and never re-reading one from HBM.
struct VtUpParams {
  const double* V;   // [n][KT] leaf bases
  const double* X;   // [n][m]
  const double* W;   // translations, heap order (node (l, i) at 2^l - 2 + i)
  double* xh;        // coefficient blocks, level-major [KT][m]
  int32_t b, m, p;
};

// C (16 x 8 NTW) = W_node^T Z for rank columns 16 mg.., columns c0..: A from W
// ([2KT][KT] row-major), B from the staged children Z (2KT rows, stride zs).
template <int KT, int NTW>
__device__ __forceinline__ void vt_up_node(const double* __restrict__ Wn, const double* Z, int zs, int mg, int c0,
                                           double* out_g, double* out_s, int m, int lane) {
  constexpr int NQ = KT / 2;  // k-steps of 4 over 2 KT rows
  constexpr int HQ = NQ < 8 ? NQ : 8;
  const int i = lane >> 2, j = lane & 3;
  const double* ap = Wn + mg * 16 + (int64_t)j * KT + 2 * i;
  const double* bp = Z + j * zs + c0 + i;
  double acc[2][NTW][2];
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt) acc[t][nt][0] = acc[t][nt][1] = 0.0;
#pragma unroll
  for (int q0 = 0; q0 < NQ; q0 += HQ) {
    double2 a[HQ];
#pragma unroll
    for (int q = 0; q < HQ; ++q) a[q] = ldg_stream2(ap + (int64_t)(q0 + q) * 4 * KT);
#pragma unroll
    for (int q = 0; q < HQ; ++q) {
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt) {
        const double bf = bp[(q0 + q) * 4 * zs + nt * 8];
        dmma(acc[0][nt][0], acc[0][nt][1], a[q].x, bf);
        dmma(acc[1][nt][0], acc[1][nt][1], a[q].y, bf);
      }
    }
  }
  store_transposed<1, NTW>(acc, out_g + (int64_t)mg * 16 * m, m, c0, m, lane);
  if (out_s) store_transposed<1, NTW>(acc, out_s + mg * 16 * zs, zs, c0, 1 << 30, lane);
}

// One up level inside the CTA: N nodes (4, 2, 1) from the 2N child blocks in
// Zin; 8 / N warps per node split MG rank groups x CS column groups.
template <int KT, int NT, int N>
__device__ __forceinline__ void vt_up_level(const VtUpParams& P, int l, int64_t n0, const double* Zin, double* Zout,
                                            int zs, int warp, int lane) {
  constexpr int MG = KT / 16, WPN = 8 / N;
  constexpr int CS0 = WPN / MG >= 1 ? WPN / MG : 1;
  constexpr int CS = CS0 < NT ? CS0 : NT;
  constexpr int NTW = NT / CS;
  const int nd = warp / WPN, sub = warp % WPN;
  if (sub >= MG * CS) return;
  const int mg = sub % MG, cs = sub / MG;
  const int64_t node = n0 + nd;
  const double* Wn = P.W + (((int64_t)1 << l) - 2 + node) * 2 * KT * KT;
  double* og = P.xh + (((int64_t)1 << l) - 2 + node) * (int64_t)KT * P.m;
  vt_up_node<KT, NTW>(Wn, Zin + (int64_t)nd * 2 * KT * zs, zs, mg, cs * NTW * 8, og,
                      Zout ? Zout + (int64_t)nd * KT * zs : nullptr, P.m, lane);
}

template <int KT, int NT>
__global__ void __launch_bounds__(256, 2) hss_vt_up_kernel(const VtUpParams P) {
  extern __shared__ double sm[];
  constexpr int MPW = KT / 16;
  constexpr int zs = NT * 8 + 4;  // rows j apart: 4 (mod 8) doubles, conflict-free B fragments
  double* L = sm;                   // 8 leaf blocks, then the 2 level-(p-2) blocks
  double* M = sm + 8 * KT * zs;     // the 4 level-(p-1) blocks
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int p = P.p, m = P.m;
  const int64_t leaf = (int64_t)blockIdx.x * 8 + warp;
  {
    double acc[2 * MPW][NT][2];
#pragma unroll
    for (int t = 0; t < 2 * MPW; ++t)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[t][nt][0] = acc[t][nt][1] = 0.0;
    warp_transposed_mma<MPW, NT, false, (MPW >= 2 ? 1 : 2)>(acc, P.V + leaf * P.b * KT, KT, P.X + leaf * P.b * m, m,
                                                            0, m, P.b, lane);
    store_transposed<MPW, NT>(acc, P.xh + (((int64_t)1 << p) - 2 + leaf) * (int64_t)KT * m, m, 0, m, lane);
    store_transposed<MPW, NT>(acc, L + warp * KT * zs, zs, 0, 1 << 30, lane);
  }
  __syncthreads();
  vt_up_level<KT, NT, 4>(P, p - 1, (int64_t)blockIdx.x * 4, L, M, zs, warp, lane);
  __syncthreads();
  vt_up_level<KT, NT, 2>(P, p - 2, (int64_t)blockIdx.x * 2, M, L, zs, warp, lane);
  __syncthreads();
  vt_up_level<KT, NT, 1>(P, p - 3, (int64_t)blockIdx.x, L, nullptr, zs, warp, lane);
}

// ---- HSS with per-level ranks, DMMA level kernels ----
// One warp = one node x one 8-row tile of its output block x one chunk of 8 NT
// columns; 8 warps per CTA. Shapes are runtime: k_l (output rows, % 8 == 0),
// the contraction lengths 2 k_{l+1} (up) and k_l, k_{l-1} (down) % 4 == 0.
// A fragments by 64-bit loads (row i of the tile, k-index 4 q + j), B fragments
// from the coefficient blocks in global memory (L2); QK k-steps of loads
// requested before their DMMAs. Same fixed summation order on every call.
struct RankedMmaParams {
  const double* G;    // up: W of level l ([2kc][k] per node); down: R of level l-1 ([2k][kp] per parent)
  const double* B;    // down: cores of the level-l siblings ([2][k][k] per pair)
  const double* xin;  // up: x of level l+1 ([kc][m] blocks); down: x of level l ([k][m])
  const double* yp;   // down: y of level l-1 ([kp][m] blocks), NULL: no parent term
  double* out;        // up: x of level l; down: y of level l ([k][m] blocks)
  int64_t nodes;      // 2^l
  int32_t k, kc, kp, m, bt;
};

// acc += A(8 rows at a0, row stride lda, or transposed: A^T with AT) . Z (K x cols at z, ld m)
template <int NT, bool AT>
__device__ __forceinline__ void ranked_tile_mma(double (&acc)[NT][2], const double* a0, int64_t lda, const double* z,
                                                int m, int K, const bool (&colok)[NT], int lane) {
  constexpr int QK = 4;
  const int i = lane >> 2, j = lane & 3;
  for (int q0 = 0; q0 < K / 4; q0 += QK) {
    double a[QK], bf[QK][NT];
#pragma unroll
    for (int u = 0; u < QK; ++u) {
      const int kk = 4 * (q0 + u) + j;
      const bool ok = 4 * (q0 + u) < K;
      a[u] = ok ? (AT ? __ldg(a0 + (int64_t)kk * lda + i) : __ldg(a0 + (int64_t)i * lda + kk)) : 0.0;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) bf[u][nt] = (ok && colok[nt]) ? ldg_cg(z + (int64_t)kk * m + nt * 8 + i) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < QK; ++u) {
      if (4 * (q0 + u) >= K) break;  // warp-uniform
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) dmma(acc[nt][0], acc[nt][1], a[u], bf[u][nt]);
    }
  }
}

template <int NT>
__device__ __forceinline__ void ranked_store(const double (&acc)[NT][2], double* out, int m, int c0, int lane) {
  const int i = lane >> 2, j = lane & 3;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int c = c0 + nt * 8 + 2 * j;
    if (c < m) out[(int64_t)i * m + c] = acc[nt][0];
    if (c + 1 < m) out[(int64_t)i * m + c + 1] = acc[nt][1];
  }
}

// One warp task of a level (defined below, shared with the cooperative sweep).
template <int NT>
__device__ __forceinline__ void ranked_up_task(const RankedMmaParams& P, int64_t gw, int lane);
template <int NT>
__device__ __forceinline__ void ranked_down_task(const RankedMmaParams& P, int64_t gw, int lane);

template <int NT>
__global__ void __launch_bounds__(256) hss_up_ranked_mma_kernel(const RankedMmaParams P) {
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (gw >= P.nodes * (P.k / 8) * ((P.m + NT * 8 - 1) / (NT * 8))) return;
  ranked_up_task<NT>(P, gw, threadIdx.x & 31);
}

template <int NT>
__global__ void __launch_bounds__(256) hss_down_ranked_mma_kernel(const RankedMmaParams P) {
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (gw >= P.nodes * (P.k / 8) * ((P.m + NT * 8 - 1) / (NT * 8))) return;
  ranked_down_task<NT>(P, gw, threadIdx.x & 31);
}

// The small levels of the per-level-rank sweeps in one cooperative launch: the
// steps (up levels, then down levels, each a RankedMmaParams) run in order with
// a grid barrier between them; inside a step the warps stride over the warp
// tasks of hss_up_ranked_mma / hss_down_ranked_mma (the same arithmetic).
constexpr int kRankedSweepMax = 2 * kMaxLevels;
struct RankedSweepParams {
  RankedMmaParams step[kRankedSweepMax];
  int32_t up[kRankedSweepMax];  // 1: upsweep step, 0: downsweep step
  int32_t nsteps;
};

// x_l[i] = W_{l,i}^T [x_{l+1}[2i]; x_{l+1}[2i+1]]   (Fig. 5 right)
template <int NT>
__device__ __forceinline__ void ranked_up_task(const RankedMmaParams& P, int64_t gw, int lane) {
  const int tiles = P.k / 8, nck = (P.m + NT * 8 - 1) / (NT * 8);
  const int64_t per = (int64_t)tiles * nck;
  const int64_t node = gw / per;
  const int rem = (int)(gw - node * per), tile = rem % tiles, c0 = (rem / tiles) * NT * 8;
  bool colok[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) colok[nt] = c0 + nt * 8 + (lane >> 2) < P.m;
  double acc[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
  ranked_tile_mma<NT, true>(acc, P.G + node * 2 * P.kc * P.k + 8 * tile, P.k,
                            P.xin + 2 * node * (int64_t)P.kc * P.m + c0, P.m, 2 * P.kc, colok, lane);
  ranked_store<NT>(acc, P.out + (node * P.k + 8 * tile) * (int64_t)P.m, P.m, c0, lane);
}

// y_l[2q+w] = S_w x_l[2q+1-w] + R_{l-1,q}[w] y_{l-1}[q]   (reading G1;
// bt: S'_w = (S_{1-w})^T, the adjoint's cores)
template <int NT>
__device__ __forceinline__ void ranked_down_task(const RankedMmaParams& P, int64_t gw, int lane) {
  const int tiles = P.k / 8, nck = (P.m + NT * 8 - 1) / (NT * 8);
  const int64_t per = (int64_t)tiles * nck;
  const int64_t jn = gw / per;
  const int rem = (int)(gw - jn * per), tile = rem % tiles, c0 = (rem / tiles) * NT * 8;
  const int64_t q = jn >> 1;
  const int w = (int)(jn & 1);
  const int k = P.k, m = P.m;
  bool colok[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) colok[nt] = c0 + nt * 8 + (lane >> 2) < m;
  double acc[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
  const double* xs = P.xin + (jn ^ 1) * (int64_t)k * m + c0;
  if (P.bt) {
    const double* S = P.B + (q * 2 + (1 - w)) * (int64_t)k * k;
    ranked_tile_mma<NT, true>(acc, S + 8 * tile, k, xs, m, k, colok, lane);
  } else {
    const double* S = P.B + (q * 2 + w) * (int64_t)k * k;
    ranked_tile_mma<NT, false>(acc, S + (int64_t)8 * tile * k, k, xs, m, k, colok, lane);
  }
  if (P.yp && P.kp > 0) {
    const double* Rn = P.G + (q * 2 * k + (int64_t)w * k) * P.kp;
    ranked_tile_mma<NT, false>(acc, Rn + (int64_t)8 * tile * P.kp, P.kp, P.yp + q * (int64_t)P.kp * m + c0, m, P.kp,
                               colok, lane);
  }
  ranked_store<NT>(acc, P.out + (jn * k + 8 * tile) * (int64_t)m, m, c0, lane);
}

template <int NT>
__global__ void __launch_bounds__(256) hss_ranked_sweep_kernel(const RankedSweepParams S) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int64_t gw0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int st = 0; st < S.nsteps; ++st) {
    if (st) grid.sync();
    const RankedMmaParams& P = S.step[st];
    const int64_t tasks = P.nodes * (P.k / 8) * ((P.m + NT * 8 - 1) / (NT * 8));
    for (int64_t gw = gw0; gw < tasks; gw += nw) {
      if (S.up[st]) ranked_up_task<NT>(P, gw, lane);
      else ranked_down_task<NT>(P, gw, lane);
    }
  }
}

}  // namespace hm
