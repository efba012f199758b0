// hm_general.cuh — general cluster trees and per-level HODLR ranks.
//
// A cluster tree of depth p is given by its leaf endpoint vector c (
// Def. 2.1): leaf i holds rows [c[i-1], c[i]) (c[-1] = 0), leaves may be
// empty (Fig. 4), and the level-l node i is the union of its 2^(p-l)
// leaves. Leaf blocks D_i are |I_i| x |I_i|, concatenated. HODLR ranks may
// differ per level ("ranks ... can vary"; the class stores one factor
// pair per block).
//
// Kernels (shape-agnostic, deterministic):
//   gen_vt_chunk   partial t = V(rows)^T X(rows) over one chunk of at most
//                  kChunkRows rows of one node (a node is split into chunks so
//                  a big top-level node is spread over many CTAs);
//   gen_vt_reduce  t_{l,j} = sum of its chunks' partials in chunk order;
//   gen_leaf       per leaf: Y(I_i) = D_i X(I_i) (or D_i^T X(I_i)) + sum_s
//                  A_s(I_i) T_s[node_s] — every level's U t_sib (HODLR) or the
//                  leaf's U y_i (HSS), Y written once.
// The HSS tree sweeps do not depend on the row partition (k x m blocks per
// node) and reuse the uniform-tree kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "hm_kernels.cuh"

namespace hm {

constexpr int64_t kChunkRows = 4096;

// One chunk: rows [lo, hi) of one node; its partial goes to partial + pidx * k * m.
struct GenChunk {
  int64_t lo, hi;
  int64_t pidx;  // global chunk index (partials are [chunks][k][m] per level group)
  int32_t lev;   // index into GenVtParams::lev
  int32_t pad;
};

struct GenVtLevel {
  const double* V;       // [n][k] right factors of this level (or HSS leaf V)
  double* out;           // [nodes][k][m]
  double* partial;       // [chunks of this level][k][m]
  const int64_t* cbeg;   // device: first chunk (relative to the level) of node j, [nodes + 1]
  int64_t nodes;
  int64_t chunk0;        // first global chunk of this level
  int32_t k;
  int32_t pad;
};

struct GenVtParams {
  const double* X;        // [n][m]
  const GenChunk* chunks; // device table, all levels
  int64_t nchunks;
  int32_t m, mc;          // columns, columns per CTA (grid.y)
  int32_t nlev;
  int32_t pad;
  GenVtLevel lev[kMaxLevels];
};

// CTA = one chunk x one column group. Thread o < O2 owns output (a = o % k,
// c = o / k); G = 256 / O2 row groups stride the chunk; fixed-order sum over
// the groups in shared memory. For k * mc > 256 threads loop over outputs.
__global__ void __launch_bounds__(kThreads) gen_vt_chunk_kernel(const GenVtParams P) {
  __shared__ double red[kThreads];
  const GenChunk ch = P.chunks[blockIdx.x];
  const GenVtLevel lv = P.lev[ch.lev];
  const int k = lv.k, m = P.m;
  const int c0 = blockIdx.y * P.mc;
  const int mc = min(P.mc, m - c0);
  const int O = k * mc;
  double* dst = lv.partial + (ch.pidx - lv.chunk0) * (int64_t)k * m;
  int O2 = 1;
  while (O2 < O) O2 <<= 1;
  if (O2 <= kThreads) {
    const int G = kThreads / O2;
    const int o = threadIdx.x % O2, g = threadIdx.x / O2;
    const int a = o % k, c = o / k;
    double acc = 0.0;
    if (o < O)
      for (int64_t r = ch.lo + g; r < ch.hi; r += G) acc = fma(lv.V[r * k + a], P.X[r * m + c0 + c], acc);
    red[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x < O) {
      double s = 0.0;
      for (int gg = 0; gg < G; ++gg) s += red[gg * O2 + threadIdx.x];
      dst[(threadIdx.x % k) * m + c0 + threadIdx.x / k] = s;
    }
  } else {
    for (int o = threadIdx.x; o < O; o += kThreads) {
      const int a = o % k, c = o / k;
      double acc = 0.0;
      for (int64_t r = ch.lo; r < ch.hi; ++r) acc = fma(lv.V[r * k + a], P.X[r * m + c0 + c], acc);
      dst[a * m + c0 + c] = acc;
    }
  }
}

// out[l][j][e] = sum_{ch = cbeg[j] .. cbeg[j+1]-1} partial[ch][e], e < k m. One
// thread per (level, node, e); levels laid out back to back (thread_begin).
struct GenReduceParams {
  int32_t nlev;
  int32_t m;
  int64_t threads;
  int64_t thread_begin[kMaxLevels + 1];
  GenVtLevel lev[kMaxLevels];
};

__global__ void __launch_bounds__(kThreads) gen_vt_reduce_kernel(const GenReduceParams P) {
  const int64_t t = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (t >= P.threads) return;
  int L = 0;
  while (L + 1 < P.nlev && P.thread_begin[L + 1] <= t) ++L;
  const GenVtLevel lv = P.lev[L];
  const int64_t km = (int64_t)lv.k * P.m;
  const int64_t local = t - P.thread_begin[L];
  const int64_t j = local / km, e = local - j * km;
  const int64_t b0 = lv.cbeg[j], b1 = lv.cbeg[j + 1];
  double s = 0.0;
  for (int64_t c = b0; c < b1; ++c) s += lv.partial[c * km + e];
  lv.out[j * km + e] = s;
}

// ------------------------------------------------------------------ leaf --

struct GenLeafParams {
  const double* D;        // concatenated |I_i| x |I_i| blocks
  const int64_t* lo;      // device [nleaves + 1]: leaf i rows [lo[i], lo[i+1])
  const int64_t* doff;    // device [nleaves]: offset of D_i
  const double* X;
  double* Y;
  int32_t m, mc;
  int32_t nseg, ktot;
  int32_t dtrans;         // 1: D_i^T (adjoint)
  int32_t pad;
  LeafSeg seg[kMaxLevels];  // node of leaf i for segment s: (i >> shift) ^ xr
};

// CTA = one leaf x one column chunk (MC = P.mc columns, MC <= kMaxMc). Z = [X(I_i);
// T_1[node_1]; ...] staged in shared memory; warp per output row, lanes striding
// the extended row, butterfly reduction (fixed order).
template <int MC>
__global__ void __launch_bounds__(kThreads) gen_leaf_kernel(const GenLeafParams P) {
  extern __shared__ double smem[];
  const int64_t leaf = blockIdx.x;
  const int64_t r0 = P.lo[leaf], b = P.lo[leaf + 1] - r0;
  if (b == 0) return;  // empty leaf: no rows
  const int c0 = blockIdx.y * MC;
  const int mc = min(MC, P.m - c0);
  double* Z = smem;  // [(b + ktot)][MC]
  for (int64_t e = threadIdx.x; e < b * MC; e += kThreads) {
    const int64_t r = e / MC;
    const int c = (int)(e - r * MC);
    Z[e] = (c < mc) ? P.X[(r0 + r) * P.m + c0 + c] : 0.0;
  }
  {
    int64_t off = b * MC;
    for (int s = 0; s < P.nseg; ++s) {
      const LeafSeg sg = P.seg[s];
      const int64_t node = (leaf >> sg.shift) ^ sg.xr;
      const double* T = sg.T + node * sg.k * P.m;
      for (int e = threadIdx.x; e < sg.k * MC; e += kThreads) {
        const int a = e / MC, c = e - a * MC;
        Z[off + e] = (c < mc) ? T[a * P.m + c0 + c] : 0.0;
      }
      off += (int64_t)sg.k * MC;
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* Di = P.D + P.doff[leaf];
  for (int64_t r = warp; r < b; r += kThreads / 32) {
    double acc[MC];
#pragma unroll
    for (int c = 0; c < MC; ++c) acc[c] = 0.0;
    for (int64_t j = lane; j < b; j += 32) {
      const double d = P.dtrans ? Di[j * b + r] : Di[r * b + j];
#pragma unroll
      for (int c = 0; c < MC; ++c) acc[c] = fma(d, Z[j * MC + c], acc[c]);
    }
    int64_t off = b;
    for (int s = 0; s < P.nseg; ++s) {
      const LeafSeg sg = P.seg[s];
      const double* Ar = sg.A + (r0 + r) * sg.k;
      for (int a = lane; a < sg.k; a += 32) {
        const double u = Ar[a];
#pragma unroll
        for (int c = 0; c < MC; ++c) acc[c] = fma(u, Z[(off + a) * MC + c], acc[c]);
      }
      off += sg.k;
    }
#pragma unroll
    for (int c = 0; c < MC; ++c) {
      double v = acc[c];
#pragma unroll
      for (int w = 16; w >= 1; w >>= 1) v += __shfl_xor_sync(0xffffffffu, v, w);
      acc[c] = v;
    }
    if (lane < mc) {
      double v = acc[0];
#pragma unroll
      for (int c = 1; c < MC; ++c)
        if (c == lane) v = acc[c];
      P.Y[(r0 + r) * P.m + c0 + lane] = v;
    }
  }
}

}  // namespace hm
