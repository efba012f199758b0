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

#include "hm_fast.cuh"

namespace hm {

constexpr int64_t kChunkRows = 4096;
#ifndef HM_GEN_MMA_Q
#define HM_GEN_MMA_Q 16  // k-steps of A fragments requested per batch in gen_leaf_mma
#endif

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
  const int32_t* order;   // execution order: CTA x runs chunk order[x] (all levels' chunks of a row
                          // range back to back, so X rows are re-read from L2, not HBM)
  int64_t nchunks;
  int32_t m, mc;          // columns, columns per CTA (grid.y)
  int32_t nlev;
  int32_t pad;
  GenVtLevel lev[kMaxLevels];
};

// nrhs = 1, k a power of two in 2..64 (hm_fast.cuh vt_gemv on a ragged chunk):
// a chunk's V rows are one contiguous run of (hi - lo) k doubles; every warp
// streams its share as 128-bit chunks (lane l keeps rank columns (2l) % k and
// (2l+1) % k, so accumulation stays in registers), x[r] from L1; butterfly
// over the lanes sharing a column, fixed-order sum over the 8 warps.
__global__ void __launch_bounds__(kThreads) gen_vt_gemv_kernel(const GenVtParams P) {
  __shared__ double red[kThreads / 32][64];
  const GenChunk ch = P.chunks[P.order[blockIdx.x]];
  const GenVtLevel lv = P.lev[ch.lev];
  const int k = lv.k;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t ne = (ch.hi - ch.lo) * k;  // doubles of the chunk (even: k even)
  const double* V = lv.V + ch.lo * k;
  const double* X = P.X + ch.lo;
  const int lk = __ffs(k) - 1;  // log2 k
  double acc0 = 0.0, acc1 = 0.0;
  constexpr int U = 4;
  for (int64_t e0 = ((int64_t)warp * 32 + lane) * 2; e0 < ne; e0 += (int64_t)kThreads * 2 * U) {
    double2 v[U];
    double x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + (int64_t)u * kThreads * 2;
      const bool ok = e < ne;
      v[u] = ok ? __ldg(reinterpret_cast<const double2*>(V + e)) : make_double2(0.0, 0.0);
      x[u] = ok ? __ldg(X + (e >> lk)) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc0 = fma(v[u].x, x[u], acc0);
      acc1 = fma(v[u].y, x[u], acc1);
    }
  }
  // lane l holds columns (2l) % k, (2l+1) % k: lanes l, l + k/2, ... share them
  for (int w = 16; w >= k / 2 && w >= 1; w >>= 1) {
    acc0 += __shfl_xor_sync(0xffffffffu, acc0, w);
    acc1 += __shfl_xor_sync(0xffffffffu, acc1, w);
  }
  if (2 * lane < k) {
    red[warp][2 * lane] = acc0;
    red[warp][2 * lane + 1] = acc1;
  }
  __syncthreads();
  if (threadIdx.x < k) {
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) sum += red[w][threadIdx.x];
    lv.partial[(ch.pidx - lv.chunk0) * (int64_t)k + threadIdx.x] = sum;
  }
}

// CTA = one chunk x one column group. Thread o < O2 owns output (a = o % k,
// c = o / k); G = 256 / O2 row groups stride the chunk; fixed-order sum over
// the groups in shared memory. For k * mc > 256 threads loop over outputs.
__global__ void __launch_bounds__(kThreads) gen_vt_chunk_kernel(const GenVtParams P) {
  __shared__ double red[kThreads];
  const GenChunk ch = P.chunks[P.order[blockIdx.x]];
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

#ifndef HM_GEN_VT_MINB
#define HM_GEN_VT_MINB 3  // CTAs per SM of the small instances (KT NT <= 16)
#endif
// nrhs >= 2, every level of rank KT in {16, 32, 64}: DMMA per chunk. Warp w
// takes an 8th of the chunk's rows (a multiple of 4), t = V(rows)^T X(rows)
// with the hm_fast.cuh fragment layout (one 128-bit load of a V row covers 16
// rank columns; rows past the chunk end read as zero), then a fixed-order sum
// over the 8 warps in shared memory. grid.y = column chunks of 8 NT.
template <int KT, int NT>
__global__ void __launch_bounds__(kThreads, KT * NT <= 16 ? HM_GEN_VT_MINB : 1) gen_vt_mma_kernel(const GenVtParams P) {
  extern __shared__ double red[];  // [8][KT][8 NT]
  constexpr int MC = NT * 8, MPW = KT / 16;
  const GenChunk ch = P.chunks[P.order[blockIdx.x]];
  const GenVtLevel lv = P.lev[ch.lev];
  const int m = P.m;
  const int c0 = blockIdx.y * MC;
  const int mc = min(MC, m - c0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = lane >> 2, j = lane & 3;
  const int64_t len = ch.hi - ch.lo;
  const int64_t slice = (len + 31) / 32 * 4;
  const int64_t r0 = ch.lo + warp * slice;
  const int64_t K = max((int64_t)0, min(ch.hi, r0 + slice) - r0);
  double acc[2 * MPW][NT][2];
#pragma unroll
  for (int t = 0; t < 2 * MPW; ++t)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[t][nt][0] = acc[t][nt][1] = 0.0;
  bool colok[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) colok[nt] = nt * 8 + i < mc;
  const double* A = lv.V + r0 * KT + 2 * i;
  const double* B = P.X + r0 * m + c0 + i;
  // batches of QB k-steps: every load of a batch issued before its DMMAs
  constexpr int QB = (MPW * NT <= 2) ? 8 : (MPW * NT <= 4 ? 4 : 2);
  int64_t q = 0;
  for (; 4 * (q + QB) <= K; q += QB) {
    double2 a[QB][MPW];
    double bf[QB][NT];
#pragma unroll
    for (int u = 0; u < QB; ++u) {
      const int64_t row = 4 * (q + u) + j;
#pragma unroll
      for (int mp = 0; mp < MPW; ++mp) a[u][mp] = __ldg(reinterpret_cast<const double2*>(A + row * KT + mp * 16));
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) bf[u][nt] = colok[nt] ? __ldg(B + row * m + nt * 8) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < QB; ++u)
#pragma unroll
      for (int mp = 0; mp < MPW; ++mp)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          dmma(acc[2 * mp][nt][0], acc[2 * mp][nt][1], a[u][mp].x, bf[u][nt]);
          dmma(acc[2 * mp + 1][nt][0], acc[2 * mp + 1][nt][1], a[u][mp].y, bf[u][nt]);
        }
  }
  if (4 * q < K) {
    // masked tail (< QB k-steps) as one batch: every load before the DMMAs
    double2 a[QB][MPW];
    double bf[QB][NT];
#pragma unroll
    for (int u = 0; u < QB; ++u) {
      const int64_t row = 4 * (q + u) + j;
      const bool ok = row < K;
#pragma unroll
      for (int mp = 0; mp < MPW; ++mp)
        a[u][mp] = ok ? __ldg(reinterpret_cast<const double2*>(A + row * KT + mp * 16)) : make_double2(0.0, 0.0);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) bf[u][nt] = (ok && colok[nt]) ? __ldg(B + row * m + nt * 8) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < QB; ++u) {
      if (4 * (q + u) >= K) break;  // warp-uniform
#pragma unroll
      for (int mp = 0; mp < MPW; ++mp)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          dmma(acc[2 * mp][nt][0], acc[2 * mp][nt][1], a[u][mp].x, bf[u][nt]);
          dmma(acc[2 * mp + 1][nt][0], acc[2 * mp + 1][nt][1], a[u][mp].y, bf[u][nt]);
        }
    }
  }
#pragma unroll
  for (int t = 0; t < 2 * MPW; ++t) {
    const int a = 16 * (t >> 1) + 2 * i + (t & 1);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      double* o = red + ((int64_t)warp * KT + a) * MC + nt * 8 + 2 * j;
      o[0] = acc[t][nt][0];
      o[1] = acc[t][nt][1];
    }
  }
  __syncthreads();
  double* dst = lv.partial + (ch.pidx - lv.chunk0) * (int64_t)KT * m;
  for (int o = threadIdx.x; o < KT * mc; o += kThreads) {
    const int a = o / mc, c = o - a * mc;
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) sum += red[((int64_t)w * KT + a) * MC + c];
    dst[a * m + c0 + c] = sum;
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
  // 8 independent running sums (chunk c goes to sum (c - b0) % 8), combined in
  // a fixed order: the loads of 8 chunks are in flight at once, and the result
  // depends only on the chunk count, never on timing
  double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  int64_t c = b0;
  for (; c + 8 <= b1; c += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] += lv.partial[(c + u) * km + e];
  }
  for (int u = 0; c < b1; ++c, ++u) acc[u] += lv.partial[c * km + e];
  const double s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  lv.out[j * km + e] = s;
}

// ------------------------------------------------------------------ leaf --

struct GenLeafParams {
  const int32_t* order;   // CTA x runs leaf order[x]: largest leaves first (shorter tail wave)
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

__host__ __device__ constexpr int gen_leaf_zs(int mc) { return mc == 1 ? 1 : mc + 2; }
// one staged row of MC doubles (16-byte aligned for MC >= 2) into registers
template <int MC>
__device__ __forceinline__ void zrow(double (&z)[MC], const double* zr) {
  if constexpr (MC == 1) {
    z[0] = zr[0];
  } else {
#pragma unroll
    for (int c = 0; c < MC; c += 2) {
      const double2 t = *reinterpret_cast<const double2*>(zr + c);
      z[c] = t.x;
      z[c + 1] = t.y;
    }
  }
}

// CTA = one leaf x one column chunk (MC = P.mc columns, MC <= kMaxMc). Z = [X(I_i);
// T_1[node_1]; ...] staged in shared memory; warp per output row, lanes striding
// the extended row, butterfly reduction (fixed order).
template <int MC>
__global__ void __launch_bounds__(kThreads) gen_leaf_kernel(const GenLeafParams P) {
  extern __shared__ double smem[];
  const int64_t leaf = P.order[blockIdx.x];
  const int64_t r0 = P.lo[leaf], b = P.lo[leaf + 1] - r0;
  if (b == 0) return;  // empty leaf: no rows
  const int c0 = blockIdx.y * MC;
  const int mc = min(MC, P.m - c0);
  // Z rows padded to ZS doubles: lanes read whole rows (jj = lane + 32 v) as
  // 128-bit loads; ZS = MC + 2 (80 B for MC = 8) puts a quarter-warp's rows in
  // distinct bank groups.
  constexpr int ZS = gen_leaf_zs(MC);
  double* Z = smem;  // [(b + ktot)][ZS]
  for (int64_t e = threadIdx.x; e < b * MC; e += kThreads) {
    const int64_t r = e / MC;
    const int c = (int)(e - r * MC);
    Z[r * ZS + c] = (c < mc) ? P.X[(r0 + r) * P.m + c0 + c] : 0.0;
  }
  {
    int64_t off = b;
    for (int s = 0; s < P.nseg; ++s) {
      const LeafSeg sg = P.seg[s];
      const int64_t node = (leaf >> sg.shift) ^ sg.xr;
      const double* T = sg.T + node * sg.k * P.m;
      for (int e = threadIdx.x; e < sg.k * MC; e += kThreads) {
        const int a = e / MC, c = e - a * MC;
        Z[(off + a) * ZS + c] = (c < mc) ? T[a * P.m + c0 + c] : 0.0;
      }
      off += sg.k;
    }
  }
  // extended-column tables of the U segments (after Z): base pointer of rank
  // column a of segment s (row 0) and the segment's row stride k
  const int kt = P.ktot;
  const double** ubase = reinterpret_cast<const double**>(Z + (b + kt) * ZS);
  int* ukst = reinterpret_cast<int*>(ubase + kt);
  {
    int e = 0;
    for (int s2 = 0; s2 < P.nseg; ++s2) {
      const int k2 = P.seg[s2].k;
      for (int a = threadIdx.x; a < k2; a += kThreads) {
        ubase[e + a] = P.seg[s2].A + a;
        ukst[e + a] = k2;
      }
      e += k2;
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* Di = P.D + P.doff[leaf];
  // A warp owns GR rows at a time (rows r0w + 8u): every lane requests GR x UJ
  // elements of D (and then of each level's U rows) before the first FMA, so
  // a warp keeps GR * UJ loads in flight instead of one (memory-level
  // parallelism for the HBM-bound leaf pass); lanes stride the columns.
  constexpr int GR = MC <= 4 ? 4 : 2;
  constexpr int UJ = 4;
  for (int64_t rw = warp; rw < b; rw += GR * (kThreads / 32)) {
    double acc[GR][MC];
#pragma unroll
    for (int u = 0; u < GR; ++u)
#pragma unroll
      for (int c = 0; c < MC; ++c) acc[u][c] = 0.0;
    bool rok[GR];
#pragma unroll
    for (int u = 0; u < GR; ++u) rok[u] = rw + 8 * u < b;
    // row pointers of the warp's rows (rows past the leaf clamp to its last
    // row: read, never stored), 32-bit column indices; only the tail chunk of
    // a row is masked
    const int bi = (int)b;
    const double* drow[GR];
#pragma unroll
    for (int u = 0; u < GR; ++u) {
      const int64_t r = rok[u] ? rw + 8 * u : b - 1;
      drow[u] = P.dtrans ? Di + r : Di + r * b;
    }
    const int64_t dstep = P.dtrans ? b : 1;  // element stride along the contraction index
    int j0 = lane;
    for (; j0 + 32 * (UJ - 1) < bi; j0 += 32 * UJ) {  // full chunks: no masks
      double d[GR][UJ];
#pragma unroll
      for (int u = 0; u < GR; ++u)
#pragma unroll
        for (int v = 0; v < UJ; ++v) d[u][v] = __ldg(drow[u] + (j0 + 32 * v) * dstep);
#pragma unroll
      for (int v = 0; v < UJ; ++v) {
        double z[MC];
        zrow<MC>(z, Z + (j0 + 32 * v) * ZS);
#pragma unroll
        for (int c = 0; c < MC; ++c)
#pragma unroll
          for (int u = 0; u < GR; ++u) acc[u][c] = fma(d[u][v], z[c], acc[u][c]);
      }
    }
    if (j0 < bi) {  // tail (< UJ chunks of 32 columns): one masked batch of loads
      double d[GR][UJ];
#pragma unroll
      for (int u = 0; u < GR; ++u)
#pragma unroll
        for (int v = 0; v < UJ; ++v) d[u][v] = (j0 + 32 * v < bi) ? __ldg(drow[u] + (j0 + 32 * v) * dstep) : 0.0;
#pragma unroll
      for (int v = 0; v < UJ; ++v) {
        if (j0 + 32 * v >= bi) break;
        double z[MC];
        zrow<MC>(z, Z + (j0 + 32 * v) * ZS);
#pragma unroll
        for (int c = 0; c < MC; ++c)
#pragma unroll
          for (int u = 0; u < GR; ++u) acc[u][c] = fma(d[u][v], z[c], acc[u][c]);
      }
    }
    // U segments, flattened: extended column e in [0, ktot) of segment s(e),
    // rank column a(e) (tables staged above). GR x UJ loads in flight per lane,
    // as for D, instead of one dependent round trip per segment.
    for (int e0 = lane; e0 < kt; e0 += 32 * UJ) {
      double uu[GR][UJ];
#pragma unroll
      for (int v = 0; v < UJ; ++v) {
        const int e = e0 + 32 * v;
        const bool eok = e < kt;
        const double* ub = eok ? ubase[e] : nullptr;
        const int ks = eok ? ukst[e] : 0;
#pragma unroll
        for (int u = 0; u < GR; ++u) uu[u][v] = (eok && rok[u]) ? __ldg(ub + (r0 + rw + 8 * u) * ks) : 0.0;
      }
#pragma unroll
      for (int v = 0; v < UJ; ++v) {
        const int e = e0 + 32 * v;
        if (e >= kt) break;
        double z[MC];
        zrow<MC>(z, Z + (b + e) * ZS);
#pragma unroll
        for (int c = 0; c < MC; ++c)
#pragma unroll
          for (int u = 0; u < GR; ++u) acc[u][c] = fma(uu[u][v], z[c], acc[u][c]);
      }
    }
#pragma unroll
    for (int u = 0; u < GR; ++u) {
#pragma unroll
      for (int c = 0; c < MC; ++c) {
        double v = acc[u][c];
#pragma unroll
        for (int w = 16; w >= 1; w >>= 1) v += __shfl_xor_sync(0xffffffffu, v, w);
        acc[u][c] = v;
      }
      if (rok[u] && lane < mc) {
        double v = acc[u][0];
#pragma unroll
        for (int c = 1; c < MC; ++c)
          if (c == lane) v = acc[u][c];
        P.Y[(r0 + rw + 8 * u) * P.m + c0 + lane] = v;
      }
    }
  }
}

// nrhs >= 2: the leaf pass on the fp64 tensor cores for any leaf size (ragged
// trees). CTA = one leaf x one chunk of 8 NT columns; Z = [X(I_i); T_1; ..]
// staged with row stride 8 NT + 4 (rows j apart: conflict-free). Warp w takes
// the leaf's 8-row tiles w, w + 8, ..; per tile the DMMA A fragments are
// D[8t + i][4q + j] (or D^T: D[4q + j][8t + i], DT) and U_s[8t + i][4q + j],
// 64-bit loads with rows / contraction indices past the block read as zero, Q
// k-steps requested before their DMMAs.
template <int NT, bool DT>
#ifndef HM_GEN_MMA_MINB
#define HM_GEN_MMA_MINB 1
#endif
__global__ void __launch_bounds__(kThreads, HM_GEN_MMA_MINB) gen_leaf_mma_kernel(const GenLeafParams P) {
  extern __shared__ double smem[];
  constexpr int MC = NT * 8, ZS = MC + 4, Q = HM_GEN_MMA_Q;
  const int64_t leaf = P.order[blockIdx.x];
  const int64_t r0 = P.lo[leaf], b = P.lo[leaf + 1] - r0;
  if (b == 0) return;
  const int c0 = blockIdx.y * MC;
  const int m = P.m, mc = min(MC, m - c0);
  double* Z = smem;  // [(b + ktot)][ZS]: X(I_i) columns c0.., then T_s[node_s] per segment (cp.async)
  stage_rows_async(Z, ZS, P.X + r0 * m + c0, m, (int)b, mc, MC);
  int64_t off = b;
  for (int s = 0; s < P.nseg; ++s) {
    const LeafSeg sg = P.seg[s];
    stage_rows_async(Z + off * ZS, ZS, sg.T + ((leaf >> sg.shift) ^ sg.xr) * sg.k * m + c0, m, sg.k, mc, MC);
    off += sg.k;
  }
  const int kt = P.ktot;
  const double** ubase = reinterpret_cast<const double**>(Z + (b + kt) * ZS);
  int* ukst = reinterpret_cast<int*>(ubase + kt);
  {
    int e = 0;
    for (int s2 = 0; s2 < P.nseg; ++s2) {
      const int k2 = P.seg[s2].k;
      for (int a2 = threadIdx.x; a2 < k2; a2 += kThreads) {
        ubase[e + a2] = P.seg[s2].A + a2;
        ukst[e + a2] = k2;
      }
      e += k2;
    }
  }
  cp_async_wait_all();
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = lane >> 2, j = lane & 3;
  const double* Di = P.D + P.doff[leaf];
  const int64_t ntile = (b + 7) / 8;
  for (int64_t t = warp; t < ntile; t += kThreads / 32) {
    const int64_t row = 8 * t + i;
    const bool rok = row < b;
    double acc[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
    // leaf block: contraction over the b columns of D_i (rows of D_i^T); rows
    // past the leaf clamp to its last row (computed, never stored); full
    // batches of Q k-steps unmasked, the tail masked
    const int bi = (int)b;
    const int64_t rr = rok ? row : b - 1;
    const double* drow = DT ? Di + rr : Di + rr * b;
    const int64_t dstep = DT ? b : 1;
    int q0 = 0;
    for (; 4 * (q0 + Q) <= bi; q0 += Q) {
      double a[Q];
#pragma unroll
      for (int u = 0; u < Q; ++u) a[u] = __ldg(drow + (4 * (q0 + u) + j) * dstep);
#pragma unroll
      for (int u = 0; u < Q; ++u) {
        const double* zr = Z + (4 * (q0 + u) + j) * ZS + i;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma(acc[nt][0], acc[nt][1], a[u], zr[nt * 8]);
      }
    }
    if (4 * q0 < bi) {
      // the tail (< Q k-steps): one masked batch, every load requested before
      // the first DMMA (a k-step at a time would expose a load latency each)
      double a[Q];
#pragma unroll
      for (int u = 0; u < Q; ++u) {
        const int kk = 4 * (q0 + u) + j;
        a[u] = kk < bi ? __ldg(drow + kk * dstep) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < Q; ++u) {
        if (4 * (q0 + u) >= bi) break;  // warp-uniform
        const int kk = 4 * (q0 + u) + j;
        const bool kok = kk < bi;
        const double* zr = Z + (kok ? kk : 0) * ZS + i;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma(acc[nt][0], acc[nt][1], a[u], kok ? zr[nt * 8] : 0.0);
      }
    }
    // U segments, flattened over the extended columns kk in [0, ktot) (tables
    // staged above): Q k-steps of A fragments U_s(kk)[row][a(kk)] requested
    // before their DMMAs, across segment boundaries
    const int64_t grow = r0 + (rok ? row : 0);
    for (int q0 = 0; 4 * q0 < kt; q0 += Q) {
      double a[Q];
#pragma unroll
      for (int u = 0; u < Q; ++u) {
        const int kk = 4 * (q0 + u) + j;
        a[u] = (rok && kk < kt) ? __ldg(ubase[kk] + grow * ukst[kk]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < Q; ++u) {
        if (4 * (q0 + u) >= kt) break;
        const int kk = 4 * (q0 + u) + j;
        const double* zr = Z + (b + (kk < kt ? kk : 0)) * ZS + i;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma(acc[nt][0], acc[nt][1], a[u], kk < kt ? zr[nt * 8] : 0.0);
      }
    }
    if (rok) {
      double* y = P.Y + (r0 + row) * m + c0;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int c = nt * 8 + 2 * j;
        if (c < mc) y[c] = acc[nt][0];
        if (c + 1 < mc) y[c + 1] = acc[nt][1];
      }
    }
  }
}

// gen_leaf_mma with 128-bit A fragments (Y = A X; the adjoint keeps the kernel
// above). A ragged leaf block D_i (b x b, any b, any offset in D) has rows that
// start on 8-byte boundaries only, so a 16-byte load of D[row][c, c+1] is legal
// only where (address of D[row][0]) / 8 + c is even. A tile's 8 rows are chosen
// to share that parity sigma — 8 consecutive rows when b is even, the rows of
// one parity of a 16-row block when b is odd (row 16 B + 2 i + par) — and the
// contraction runs over columns sigma + 8 g + [0, 8) in groups: lane (i, j)
// loads D[row_i][sigma + 8 g + 2 j, + 1] (one LDG.128: ".x" feeds k-step 2 g,
// ".y" k-step 2 g + 1, B rows sigma + 8 g + 2 j (+ 1) of the staged Z — the
// k-permutation of warp_rowmajor_mma). The columns left over (column 0 when
// sigma = 1, the < 8 after the last group) form two masked 64-bit k-steps.
// U segments with k % 8 == 0 and a 16-byte aligned base stream the same way
// (8-column groups, flattened over the segments through a group table); the
// others fall back to 64-bit fragments per extended column.
// Shared memory: Z [(smax + ktot)][ZS], ZS = 8 NT + 2 (rows 2 j apart:
// conflict-free 64-bit B fragments), then the group table (pointer, row stride,
// Z row) and the per-column table of the fallback segments.
#ifndef HM_GEN_AL_QG
#define HM_GEN_AL_QG 8  // 8-column groups per batch of loads
#endif
#ifndef HM_GEN_AL_MINB
#define HM_GEN_AL_MINB 3  // CTAs per SM for NT = 1
#endif
__host__ __device__ constexpr int gen_al_zs(int nt) { return 8 * nt + 2; }
__host__ __device__ constexpr size_t gen_al_tab_bytes(int ktot) { return 32 * (size_t)ktot + 64; }

template <int NT>
__global__ void __launch_bounds__(kThreads, NT == 1 ? HM_GEN_AL_MINB : 1) gen_leaf_mma_al_kernel(const GenLeafParams P) {
  extern __shared__ double smem[];
  constexpr int MC = NT * 8, ZS = gen_al_zs(NT), QG = HM_GEN_AL_QG;  // 8-column groups per batch of loads
  const int64_t leaf = P.order[blockIdx.x];
  const int64_t r0 = P.lo[leaf], b = P.lo[leaf + 1] - r0;
  if (b == 0) return;
  const int c0 = blockIdx.y * MC;
  const int m = P.m, mc = min(MC, m - c0);
  double* Z = smem;  // [(b + ktot)][ZS]: X(I_i) columns c0.., then T_s[node_s] per segment (cp.async)
  stage_rows_async(Z, ZS, P.X + r0 * m + c0, m, (int)b, mc, MC);
  {
    int64_t off = b;
    for (int s = 0; s < P.nseg; ++s) {
      const LeafSeg sg = P.seg[s];
      stage_rows_async(Z + off * ZS, ZS, sg.T + ((leaf >> sg.shift) ^ sg.xr) * sg.k * m + c0, m, sg.k, mc, MC);
      off += sg.k;
    }
  }
  // tables: groups of 8 rank columns of the 128-bit segments, single columns of the others
  const int kt = P.ktot;
  const double** gbase = reinterpret_cast<const double**>(Z + (b + kt) * ZS);
  const double** sbase = gbase + (kt / 8 + 1);
  int* gk = reinterpret_cast<int*>(sbase + kt + 1);
  int* gz = gk + (kt / 8 + 1);
  int* sk = gz + (kt / 8 + 1);
  int* sz = sk + kt + 1;
  int ng = 0, ns = 0;  // every thread derives the counts (same loop, no synchronisation needed)
  {
    int zrow = (int)b;
    for (int s2 = 0; s2 < P.nseg; ++s2) {
      const LeafSeg sg = P.seg[s2];
      const bool wide = (sg.k % 8 == 0) && ((reinterpret_cast<uintptr_t>(sg.A) & 15) == 0);
      if (wide) {
        for (int g = threadIdx.x; g < sg.k / 8; g += kThreads) {
          gbase[ng + g] = sg.A + 8 * g;
          gk[ng + g] = sg.k;
          gz[ng + g] = zrow + 8 * g;
        }
        ng += sg.k / 8;
      } else {
        for (int a2 = threadIdx.x; a2 < sg.k; a2 += kThreads) {
          sbase[ns + a2] = sg.A + a2;
          sk[ns + a2] = sg.k;
          sz[ns + a2] = zrow + a2;
        }
        ns += sg.k;
      }
      zrow += sg.k;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = lane >> 2, j = lane & 3;
  const double* Di = P.D + P.doff[leaf];
  const bool bodd = (b & 1) != 0;
  const int64_t ntile = bodd ? 2 * ((b + 15) / 16) : (b + 7) / 8;
  const int bi = (int)b;
  // the first batch of D loads of the warp's first tile is requested before the
  // staging wait: the row addresses need no staged data
  double2 a[QG];  // the A-fragment batch buffer (first batch filled before the wait)
  bool pre = false;
  if (warp < ntile) {
    const int64_t t = warp;
    const int64_t row0 = bodd ? 16 * (t >> 1) + (t & 1) : 8 * t;
    if (row0 < b) {
      const int64_t row = bodd ? row0 + 2 * i : row0 + i;
      const double* drow = Di + (row < b ? row : row0) * b;
      const int sig = (int)((reinterpret_cast<uintptr_t>(Di + row0 * b) >> 3) & 1);
      const int G = (bi - sig) / 8;
#pragma unroll
      for (int u = 0; u < QG; ++u) a[u] = u < G ? ld_a_stream2(drow + sig + 2 * j + 8 * u) : make_double2(0.0, 0.0);
      pre = true;
    }
  }
  cp_async_wait_all();
  __syncthreads();
  for (int64_t t = warp; t < ntile; t += kThreads / 32) {
    const int64_t row0 = bodd ? 16 * (t >> 1) + (t & 1) : 8 * t;
    if (row0 >= b) continue;  // warp-uniform: a parity tile past the block
    const int64_t row = bodd ? row0 + 2 * i : row0 + i;
    const bool rok = row < b;
    const int64_t rr = rok ? row : row0;  // same parity as the tile's rows
    const double* drow = Di + rr * b;
    const int sig = (int)((reinterpret_cast<uintptr_t>(Di + row0 * b) >> 3) & 1);
    double acc[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
    // full groups of 8 aligned columns: lane (i, j) loads D[row][sigma + 8 g + 2 j, + 1]
    const int G = (bi - sig) / 8;
    const double* da = drow + sig + 2 * j;
    const double* zb = Z + (int64_t)(sig + 2 * j) * ZS + i;
    for (int g0 = 0; g0 < G; g0 += QG) {
      if (!pre) {  // warp-uniform (pre: this batch was requested before the staging wait)
#pragma unroll
        for (int u = 0; u < QG; ++u) a[u] = (g0 + u < G) ? ld_a_stream2(da + 8 * (g0 + u)) : make_double2(0.0, 0.0);
      }
      pre = false;
#pragma unroll
      for (int u = 0; u < QG; ++u) {
        if (g0 + u >= G) break;  // warp-uniform
        const double* zr = zb + (int64_t)(8 * (g0 + u)) * ZS;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma(acc[nt][0], acc[nt][1], a[u].x, zr[nt * 8]);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma(acc[nt][0], acc[nt][1], a[u].y, zr[ZS + nt * 8]);
      }
    }
    pre = false;  // (G == 0: the prefetched batch was all zeros)
    // leftover columns: 0 (sigma = 1) and [sigma + 8 G, b): at most 8, two masked k-steps
    {
      const int nrem = bi - 8 * G;  // = sig + (b - sig - 8 G)
      double a2[2];
      int col[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int sl = 4 * u + j;
        col[u] = (sig && sl == 0) ? 0 : 8 * G + sl;  // sigma = 1: slot 0 is column 0, slot s > 0 column 8 G + s
        a2[u] = sl < nrem ? drow[col[u]] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (4 * u >= nrem) break;  // warp-uniform
        const bool ok = 4 * u + j < nrem;
        const double* zr = Z + (int64_t)(ok ? col[u] : 0) * ZS + i;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma(acc[nt][0], acc[nt][1], a2[u], ok ? zr[nt * 8] : 0.0);
      }
    }
    // U segments, 128-bit groups (flattened over the segments)
    const int64_t grow = r0 + rr;
    for (int g0 = 0; g0 < ng; g0 += QG) {
#pragma unroll
      for (int u = 0; u < QG; ++u)
        a[u] = (g0 + u < ng) ? ld_a_stream2(gbase[g0 + u] + grow * gk[g0 + u] + 2 * j) : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < QG; ++u) {
        if (g0 + u >= ng) break;
        const double* zr = Z + (int64_t)(gz[g0 + u] + 2 * j) * ZS + i;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma(acc[nt][0], acc[nt][1], a[u].x, zr[nt * 8]);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma(acc[nt][0], acc[nt][1], a[u].y, zr[ZS + nt * 8]);
      }
    }
    // U segments with 64-bit fragments (k % 8 != 0 or an unaligned base)
    for (int q0 = 0; 4 * q0 < ns; q0 += QG) {
      double as[QG];
#pragma unroll
      for (int u = 0; u < QG; ++u) {
        const int kk = 4 * (q0 + u) + j;
        as[u] = kk < ns ? __ldg(sbase[kk] + grow * sk[kk]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < QG; ++u) {
        if (4 * (q0 + u) >= ns) break;
        const int kk = 4 * (q0 + u) + j;
        const double* zr = Z + (int64_t)(kk < ns ? sz[kk] : 0) * ZS + i;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma(acc[nt][0], acc[nt][1], as[u], kk < ns ? zr[nt * 8] : 0.0);
      }
    }
    if (rok) {
      double* y = P.Y + (r0 + row) * m + c0;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int c = nt * 8 + 2 * j;
        if (c < mc) y[c] = acc[nt][0];
        if (c + 1 < mc) y[c + 1] = acc[nt][1];
      }
    }
  }
}

}  // namespace hm
