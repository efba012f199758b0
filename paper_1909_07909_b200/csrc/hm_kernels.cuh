// hm_kernels.cuh — sm_100a kernels for the HODLR / HSS matvec hot path.
//
// Paper: hm-toolbox (arXiv 1909.07909), PAPER.md "P:n" = line n.
// Three kernel families cover every step of both products:
//
//   vt_contract  t_{l,j} = V_l(I_j)^T X(I_j) for several levels in ONE pass
//                over the row tiles of X (X tile staged in shared memory and
//                reused across levels). HODLR: the V12^* v2 / V21^* v1 halves
//                of "y2 <- A12 v2", "y3 <- A21 v1" (Fig. 5 left),
//                all levels at once because HODLR blocks are independent
//                across levels. HSS: Step 1, v_i^p = V_i^* v(I_i)
//                (P:684-686). Nodes larger than a tile leave per-tile
//                partials, summed by reduce_partials in a fixed order.
//   leaf_apply   per leaf i: Y(I_i) = D_i X(I_i) + sum_s U_s(I_i) T_s[node_s]
//                with Y written exactly once. HODLR: "if A is dense return Av"
//                 plus every level's U (V^* v) term (y1+y2 / y3+y4,
//                P:674-675). HSS: Step 4, y = U_i v_i^p + d_i.
//   hss_up_level / hss_down_level
//                level-synchronous batched k x k products: upsweep through
//                R_V^* = W^T and, fused, coupling by the cores B
//                (reading G1) + downsweep through R_U.
//
// All arithmetic fp64. No atomics: every output element has one owner and a
// fixed summation order, so results are bitwise reproducible.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hm {

constexpr int kThreads = 256;
constexpr int kMaxLevels = 48;
constexpr int kMaxRank = 64;

// ----------------------------------------------------------- vt_contract --

struct VtLevel {
  const double* V;  // [n][k] rows of this level's right factors
  double* out;      // complete node results  [nodes][k][m]
  double* partial;  // per-tile partials       [n / tile][k][m] (nodes larger than a tile)
  int64_t s;        // node size (rows); s % tile == 0 or tile % s == 0
  int32_t k;
  int32_t pad;
};

struct VtParams {
  const double* X;  // [n][m]
  int64_t n;
  int32_t m;
  int32_t mc;       // columns per CTA (grid.y = ceil(m / mc))
  int64_t tile;     // rows per CTA (a whole number of leaves)
  int32_t nlev;
  VtLevel lev[kMaxLevels];
};

// One CTA = one row tile x one column chunk; loops over the levels.
// Thread t owns output o = t % O2 of the (k x mc) block (a = o % k, c = o / k)
// for the rows r == t / O2 (mod 256 / O2) of the current segment, then a
// fixed-order shared-memory reduction over the row groups.
static __global__ void __launch_bounds__(kThreads) vt_contract_kernel(const VtParams P) {
  extern __shared__ double smem[];
  const int64_t tile = P.tile;
  const int64_t row0 = (int64_t)blockIdx.x * tile;
  const int c0 = blockIdx.y * P.mc;
  const int mc = min(P.mc, P.m - c0);
  double* Xs = smem;                       // [tile][mc]
  double* red = smem + tile * P.mc;        // [kThreads]
  for (int64_t e = threadIdx.x; e < tile * mc; e += kThreads) {
    int64_t r = e / mc;
    int c = (int)(e - r * mc);
    Xs[r * mc + c] = P.X[(row0 + r) * P.m + c0 + c];
  }
  __syncthreads();
  for (int L = 0; L < P.nlev; ++L) {
    const VtLevel lv = P.lev[L];
    const int k = lv.k;
    if (k == 0) continue;
    const int O = k * mc;
    int O2 = 1;
    while (O2 < O) O2 <<= 1;
    const bool big = lv.s > tile;       // node spans several tiles: per-tile partials
    const int64_t seglen = big ? tile : lv.s;
    const int64_t nseg = tile / seglen;
    if (O2 <= kThreads) {
      const int G = kThreads / O2;
      const int o = threadIdx.x % O2, g = threadIdx.x / O2;
      const int a = o % k, c = o / k;
      for (int64_t sgi = 0; sgi < nseg; ++sgi) {
        const int64_t rb = sgi * seglen;
        double acc = 0.0;
        if (o < O) {
          const double* Vp = lv.V + (row0 + rb) * k + a;
          const double* Xp = Xs + rb * mc + c;
          for (int64_t r = g; r < seglen; r += G) acc = fma(Vp[r * k], Xp[r * mc], acc);
        }
        red[threadIdx.x] = acc;
        __syncthreads();
        if (threadIdx.x < O) {
          double s = 0.0;
          for (int gg = 0; gg < G; ++gg) s += red[gg * O2 + threadIdx.x];
          const int aa = threadIdx.x % k, cc = threadIdx.x / k;
          double* dst;
          if (big) {
            dst = lv.partial + (int64_t)blockIdx.x * k * P.m;
          } else {
            const int64_t node = (row0 + rb) / lv.s;
            dst = lv.out + node * k * P.m;
          }
          dst[aa * P.m + c0 + cc] = s;
        }
        __syncthreads();
      }
    } else {
      for (int64_t sgi = 0; sgi < nseg; ++sgi) {
        const int64_t rb = sgi * seglen;
        for (int o = threadIdx.x; o < O; o += kThreads) {
          const int a = o % k, c = o / k;
          const double* Vp = lv.V + (row0 + rb) * k + a;
          const double* Xp = Xs + rb * mc + c;
          double acc = 0.0;
          for (int64_t r = 0; r < seglen; ++r) acc = fma(Vp[r * k], Xp[r * mc], acc);
          double* dst;
          if (big) {
            dst = lv.partial + (int64_t)blockIdx.x * k * P.m;
          } else {
            const int64_t node = (row0 + rb) / lv.s;
            dst = lv.out + node * k * P.m;
          }
          dst[a * P.m + c0 + c] = acc;
        }
      }
    }
  }
}

// t_l[node] = sum_{j < s/tile} partial_l[node * (s/tile) + j] in a fixed order
// that depends only on the shapes, never on timing. Two mappings, chosen per
// level (each level owns a range of CTAs, block_begin):
//  * mode 0 (k m < 32): a group of G = 2^log2g consecutive lanes owns one output;
//    lane g sums j = g, g+G, ... (8 running sums), then a butterfly over the group;
//  * mode 1 (k m a multiple of 32): a warp owns 32 consecutive outputs of one
//    node (coalesced loads of every partial row), W = 2^log2g warps split the
//    partials j = w, w+W, ... (8 running sums each), and the W warp sums are
//    added in warp order through shared memory;
//  * mode 2 (k m < 32, >= 512 partials per node, e.g. config 5's top levels): a CTA per
//    output, the 256 threads' sums combined by warp butterflies and warp order.
struct ReduceLevel {
  const double* partial;
  double* out;
  int64_t nodes;
  int64_t block_begin;  // first CTA of this level
  int32_t per_node;     // tiles per node
  int32_t km;           // k * m
  int32_t log2g;        // mode 0: lanes per output; mode 1: warps per 32 outputs
  int32_t mode;
};
struct ReduceParams {
  int32_t nlev;
  int64_t blocks;
  ReduceLevel lev[kMaxLevels];
};

__device__ __forceinline__ double strided_sum8(const double* src, int64_t stride, int j, int step, int count) {
  double r[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  for (; j + 7 * step < count; j += 8 * step) {
#pragma unroll
    for (int u = 0; u < 8; ++u) r[u] += src[(int64_t)(j + u * step) * stride];
  }
  // the < 8 remaining partials, in order, through an unrolled guard (a
  // register array indexed at run time would live in local memory)
#pragma unroll
  for (int u = 0; u < 7; ++u)
    if (j + u * step < count) r[u] += src[(int64_t)(j + u * step) * stride];
  return ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
}

static __global__ void __launch_bounds__(kThreads) reduce_partials_kernel(const ReduceParams P) {
  __shared__ double red[kThreads];
  int L = 0;
  while (L + 1 < P.nlev && P.lev[L + 1].block_begin <= (int64_t)blockIdx.x) ++L;
  const ReduceLevel lv = P.lev[L];
  const int64_t blk = (int64_t)blockIdx.x - lv.block_begin;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lv.mode == 0) {
    const int64_t local = blk * kThreads + threadIdx.x;
    const int G = 1 << lv.log2g;
    const int64_t oi = local >> lv.log2g;
    const int g = (int)(local & (G - 1));
    const bool active = oi < lv.nodes * lv.km;
    double s = 0.0;
    if (active) {
      const int64_t node = oi / lv.km;
      const int64_t o = oi - node * lv.km;
      const double* src = lv.partial + node * (int64_t)lv.per_node * lv.km + o;
      double r[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      int j = g;
      for (; j + 7 * G < lv.per_node; j += 8 * G) {
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] += src[(int64_t)(j + u * G) * lv.km];
      }
      for (int u = 0; j < lv.per_node; j += G, ++u) r[u] += src[(int64_t)j * lv.km];
      s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    }
    for (int w = 1; w < 32; w <<= 1)
      if (w < G) s += __shfl_xor_sync(0xffffffffu, s, w);
    if (active && g == 0) lv.out[oi] = s;
    return;
  }
  if (lv.mode == 2) {
    // one CTA per output (very long sums, few outputs): thread t sums j = t,
    // t + 256, ...; then a butterfly per warp and the 8 warp sums in warp order
    const int64_t oi = blk;
    const int64_t node = oi / lv.km;
    const int64_t o = oi - node * lv.km;
    double s = strided_sum8(lv.partial + node * (int64_t)lv.per_node * lv.km + o, lv.km, threadIdx.x, kThreads,
                            lv.per_node);
    for (int w = 16; w >= 1; w >>= 1) s += __shfl_xor_sync(0xffffffffu, s, w);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = red[0];
      for (int u = 1; u < kThreads / 32; ++u) t += red[u];
      lv.out[oi] = t;
    }
    return;
  }
  const int W = 1 << lv.log2g;              // warps per slab of 32 outputs
  const int64_t slab = blk * (kThreads / 32 / W) + warp / W;
  const int sub = warp & (W - 1);
  const int64_t oi = slab * 32 + lane;      // k m % 32 == 0: a slab lies in one node
  const bool active = oi < lv.nodes * lv.km;
  double s = 0.0;
  if (active) {
    const int64_t node = oi / lv.km;
    const int64_t o = oi - node * lv.km;
    s = strided_sum8(lv.partial + node * (int64_t)lv.per_node * lv.km + o, lv.km, sub, W, lv.per_node);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  if (active && sub == 0) {
    double t = red[threadIdx.x];
    for (int u = 1; u < W; ++u) t += red[threadIdx.x + 32 * u];
    lv.out[oi] = t;
  }
}

// Distributed HODLR: after the allgather of every rank's
// partial top-level products t_l^(r) = V_l(I_r)^T X(I_r), rank `rank` needs
// t_{l, sib} = sum of the partials of the ranks under the sibling of its
// level-l ancestor, summed in increasing rank order (fixed order).
struct CombineParams {
  const double* gathered;  // [P][per_rank]
  double* out;             // [per_rank]
  int64_t per_rank;        // sum_{l <= q} k_l m
  int32_t q, rank;
  int64_t lev_off[kMaxLevels + 2];  // start of level l's block (l = 1..q), lev_off[q+1] = per_rank
};

static __global__ void __launch_bounds__(kThreads) dist_combine_kernel(const CombineParams C) {
  const int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (e >= C.per_rank) return;
  int l = 1;
  while (l < C.q && C.lev_off[l + 1] <= e) ++l;
  const int a = C.rank >> (C.q - l);
  const int span = 1 << (C.q - l);
  const int r0 = (a ^ 1) * span;
  double s = 0.0;
  for (int r = r0; r < r0 + span; ++r) s += C.gathered[(int64_t)r * C.per_rank + e];
  C.out[e] = s;
}

// Distributed HODLR with the exchange overlapped (hodlr_matvec_dist): the leaf
// pass runs while the allgather is in flight with the subtree levels only, and
// the q top-level terms Y(I_r) += sum_{l <= q} U_l(I_r) t_l (Fig. 5 left's
// y1 + y2 / y3 + y4 for the levels whose sibling block lives on other ranks,
// P:666-678) are added afterwards. Thread per (row, column); fixed order.
struct TopEpilogueParams {
  double* Y;
  const double* U;  // the rank's U_local (level-major)
  const double* T;  // packed [sum_{l<=q} k_l][m] coefficient blocks (dist_combine output)
  int64_t n;
  int32_t m, nlev, ktot, pad;
  int32_t k[kMaxLevels];
  int64_t uoff[kMaxLevels];
};

static __global__ void __launch_bounds__(kThreads) dist_top_epilogue_kernel(const TopEpilogueParams P) {
  extern __shared__ double ts[];  // T staged: ktot * m doubles
  for (int i = threadIdx.x; i < P.ktot * P.m; i += blockDim.x) ts[i] = P.T[i];
  __syncthreads();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= P.n * P.m) return;
  const int64_t r = e / P.m;
  const int c = (int)(e - r * P.m);
  double acc = 0.0;
  int toff = 0;
  for (int l = 0; l < P.nlev; ++l) {
    const double* u = P.U + P.uoff[l] + r * P.k[l];
    for (int a = 0; a < P.k[l]; ++a) acc = fma(u[a], ts[(toff + a) * P.m + c], acc);
    toff += P.k[l];
  }
  P.Y[e] += acc;
}

// ------------------------------------------------------------ leaf_apply --

struct LeafSeg {
  const double* A;  // [n][k]: this term's left factor rows (U_l or HSS U)
  const double* T;  // coefficient blocks [nodes][k][m]
  int32_t k;
  int32_t shift;    // node = (leaf >> shift) ^ xr
  int32_t xr;
  int32_t pad;
};
struct LeafParams {
  const double* D;  // [nleaves][b][b]
  const double* X;  // [n][m]
  double* Y;        // [n][m]
  int64_t b;
  int32_t m;
  int32_t mc;       // columns per CTA
  int32_t nseg;
  int32_t ktot;     // sum of segment ranks
  int32_t dtrans;   // 1: the leaf term is D_i^T X(I_i) (adjoint product)
  LeafSeg seg[kMaxLevels];
};

constexpr int kMaxMc = 16;

// One CTA = one leaf x one column chunk. The CTA stages the "extended" right
// operand Z = [X(I_i); T_1[node_1]; ...; T_S[node_S]] ((b + sum k) x mc) in
// shared memory; each warp then owns rows r of the leaf and computes
// Y[r][c] = [D_i[r][:], U_1[r][:], ..., U_S[r][:]] . Z[:][c] with lanes
// striding the extended row, then a butterfly reduction.
template <int MC>
__global__ void __launch_bounds__(kThreads) leaf_apply_kernel(const LeafParams P) {
  extern __shared__ double smem[];
  const int64_t leaf = blockIdx.x;
  const int64_t b = P.b;
  const int64_t r0 = leaf * b;
  const int c0 = blockIdx.y * MC;
  const int mc = min(MC, P.m - c0);
  double* Z = smem;  // [(b + ktot)][MC]
  for (int64_t e = threadIdx.x; e < b * MC; e += kThreads) {
    int64_t r = e / MC;
    int c = (int)(e - r * MC);
    Z[e] = (c < mc) ? P.X[(r0 + r) * P.m + c0 + c] : 0.0;
  }
  {
    int64_t off = b * MC;
    for (int s = 0; s < P.nseg; ++s) {
      const LeafSeg sg = P.seg[s];
      const int64_t node = (leaf >> sg.shift) ^ sg.xr;
      const double* T = sg.T + node * sg.k * P.m;
      for (int e = threadIdx.x; e < sg.k * MC; e += kThreads) {
        int a = e / MC, c = e - a * MC;
        Z[off + e] = (c < mc) ? T[a * P.m + c0 + c] : 0.0;
      }
      off += (int64_t)sg.k * MC;
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* Di = P.D + leaf * b * b;
  for (int64_t r = warp; r < b; r += kThreads / 32) {
    double acc[MC];
#pragma unroll
    for (int c = 0; c < MC; ++c) acc[c] = 0.0;
    const double* Dr = Di + r * b;
    for (int64_t j = lane; j < b; j += 32) {
      const double d = P.dtrans ? Di[j * b + r] : Dr[j];  // D_i^T: column r of D_i
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

// ------------------------------------------------------------------- HSS --

// Upsweep, one level l:  x_l[i] = W_{l,i}^T [x_{l+1}[2i]; x_{l+1}[2i+1]]
// W node (l,i) at index 2^l - 2 + i, [2k][k]. x level l at node offset 2^l - 2.
struct HssLevelParams {
  const double* W;   // or R for the downsweep
  const double* B;
  double* xh;        // [(2^{p+1}-2)][k][m]
  double* yh;
  const double* R_root;  // optional subtree-root term at level 1 (distributed HSS)
  const double* y_root;
  int32_t level;
  int32_t k;
  int32_t m;
  int32_t bt;        // 1: cores of the adjoint, S'_0 = B21^T, S'_1 = B12^T
};

static __global__ void __launch_bounds__(kThreads) hss_up_level_kernel(const HssLevelParams P) {
  const int l = P.level, k = P.k, m = P.m;
  const int64_t cnt = 1ll << l;
  const int64_t km = (int64_t)k * m;
  const int64_t total = cnt * km;
  for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < total; e += (int64_t)gridDim.x * kThreads) {
    const int64_t i = e / km;
    const int o = (int)(e - i * km);
    const int a = o / m, c = o - a * m;
    const double* Wn = P.W + ((1ll << l) - 2 + i) * 2 * k * k;
    const double* z0 = P.xh + ((1ll << (l + 1)) - 2 + 2 * i) * km;
    const double* z1 = z0 + km;
    double acc = 0.0;
    for (int r = 0; r < k; ++r) acc = fma(Wn[r * k + a], z0[r * m + c], acc);
    for (int r = 0; r < k; ++r) acc = fma(Wn[(k + r) * k + a], z1[r * m + c], acc);
    P.xh[((1ll << l) - 2 + i) * km + o] = acc;
  }
}

// Coupling + downsweep, one level l = 1..p (reading G1):
//   y_l[2q+w] = S_w x_l[2q+1-w] + (l >= 2 ? R_{l-1,q}[w] y_{l-1}[q] : 0)
// S_0 = B12, S_1 = B21 of node (l-1, q) (index 2^{l-1}-1+q); R node (l-1,q)
// at index 2^{l-1}-2+q, rows w*k..w*k+k-1.
static __global__ void __launch_bounds__(kThreads) hss_down_level_kernel(const HssLevelParams P) {
  const int l = P.level, k = P.k, m = P.m;
  const int64_t cnt = 1ll << l;
  const int64_t km = (int64_t)k * m;
  const int64_t total = cnt * km;
  for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < total; e += (int64_t)gridDim.x * kThreads) {
    const int64_t j = e / km;
    const int o = (int)(e - j * km);
    const int a = o / m, c = o - a * m;
    const int64_t q = j >> 1;
    const int w = (int)(j & 1);
    const double* xs = P.xh + ((1ll << l) - 2 + (j ^ 1)) * km;
    double yc = 0.0;
    if (P.bt) {  // S'_w = (S_{1-w})^T
      const double* S = P.B + (((1ll << (l - 1)) - 1 + q) * 2 + (1 - w)) * k * k;
      for (int r = 0; r < k; ++r) yc = fma(S[r * k + a], xs[r * m + c], yc);
    } else {
      const double* S = P.B + (((1ll << (l - 1)) - 1 + q) * 2 + w) * k * k;
      for (int r = 0; r < k; ++r) yc = fma(S[a * k + r], xs[r * m + c], yc);
    }
    double yd = 0.0;
    if (l >= 2) {
      const double* Rn = P.W + (((1ll << (l - 1)) - 2 + q) * 2 * k + w * k) * k;
      const double* yp = P.yh + ((1ll << (l - 1)) - 2 + q) * km;
      for (int r = 0; r < k; ++r) yd = fma(Rn[a * k + r], yp[r * m + c], yd);
    } else if (P.R_root) {
      const double* Rn = P.R_root + (int64_t)w * k * k;
      for (int r = 0; r < k; ++r) yd = fma(Rn[a * k + r], P.y_root[r * m + c], yd);
    }
    P.yh[((1ll << l) - 2 + j) * km + o] = yc + yd;
  }
}

// ------------------------------------------------ HSS, per-level ranks --
// k_l columns on level l (2k_{l+1} x k_l translations, k_l x k_l cores).
// One launch per level, thread per output entry, fixed-order sums (the generic
// kernels above with the child / parent ranks separated).
struct HssRankedLevelParams {
  const double* G;    // up: W of level l (node i at i 2 kc k); down: R of level l-1 (node q at q 2 k kp)
  const double* B;    // down: cores of the level-l siblings (pair q at q 2 k^2)
  const double* xin;  // up: x of level l+1 (kc x m blocks); down: x of level l (k x m)
  const double* yp;   // down: y of level l-1 (kp x m blocks), NULL on level 1
  double* out;        // up: x of level l; down: y of level l
  int32_t l, k, kc, kp, m, bt;
};

// x_l[i] = W_{l,i}^T [x_{l+1}[2i]; x_{l+1}[2i+1]]   (Fig. 5 right)
static __global__ void __launch_bounds__(kThreads) hss_up_ranked_kernel(const HssRankedLevelParams P) {
  const int k = P.k, kc = P.kc, m = P.m;
  const int64_t km = (int64_t)k * m, total = (1ll << P.l) * km;
  for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < total; e += (int64_t)gridDim.x * kThreads) {
    const int64_t i = e / km;
    const int o = (int)(e - i * km);
    const int a = o / m, c = o - a * m;
    const double* Wn = P.G + i * 2 * kc * k;
    const double* z0 = P.xin + 2 * i * kc * m;
    const double* z1 = z0 + (int64_t)kc * m;
    double acc = 0.0;
    for (int r = 0; r < kc; ++r) acc = fma(Wn[r * k + a], z0[r * m + c], acc);
    for (int r = 0; r < kc; ++r) acc = fma(Wn[(kc + r) * k + a], z1[r * m + c], acc);
    P.out[e] = acc;
  }
}

// y_l[2q+w] = S_w x_l[2q+1-w] + R_{l-1,q}[w] y_{l-1}[q]   (reading G1)
static __global__ void __launch_bounds__(kThreads) hss_down_ranked_kernel(const HssRankedLevelParams P) {
  const int k = P.k, kp = P.kp, m = P.m;
  const int64_t km = (int64_t)k * m, total = (1ll << P.l) * km;
  for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < total; e += (int64_t)gridDim.x * kThreads) {
    const int64_t j = e / km;
    const int o = (int)(e - j * km);
    const int a = o / m, c = o - a * m;
    const int64_t q = j >> 1;
    const int w = (int)(j & 1);
    const double* xs = P.xin + (j ^ 1) * km;
    double yc = 0.0;
    if (P.bt) {  // S'_w = (S_{1-w})^T (adjoint)
      const double* S = P.B + (q * 2 + (1 - w)) * k * k;
      for (int r = 0; r < k; ++r) yc = fma(S[r * k + a], xs[r * m + c], yc);
    } else {
      const double* S = P.B + (q * 2 + w) * k * k;
      for (int r = 0; r < k; ++r) yc = fma(S[a * k + r], xs[r * m + c], yc);
    }
    double yd = 0.0;
    if (P.yp && kp > 0) {
      const double* Rn = P.G + (q * 2 * k + w * k) * kp;
      const double* y0 = P.yp + q * (int64_t)kp * m;
      for (int r = 0; r < kp; ++r) yd = fma(Rn[a * kp + r], y0[r * m + c], yd);
    }
    P.out[e] = yc + yd;
  }
}

// ------------------------------------------ HSS, per-node ranks (padding) --
// Per-node ranks run on the per-level layout with K_l = the level's
// largest rank: every compact generator block is copied into the top-left
// corner of its zero-filled padded block (an exact embedding: the padded
// rows / columns are zero). CTA per block, threads over its elements.
struct PadBlock {
  int64_t src, dst;     // element offsets (source array / destination array)
  int32_t rows, cols;   // compact block (0 x 0: an all-zero padded block)
  int32_t drows, dcols; // padded block; destination row stride = dcols
  int32_t arr, pad;     // array id (0 U, 1 V, 2 R, 3 W, 4 B)
};
struct PadParams {
  const PadBlock* blocks;
  const double* src[5];
  double* dst[5];
};

// Writes every element of one padded block exactly once: the compact block
// in its top-left corner, zeros elsewhere.
static __global__ void __launch_bounds__(kThreads) pad_blocks_kernel(const PadParams P, int64_t nblocks) {
 for (int64_t bi = blockIdx.x; bi < nblocks; bi += gridDim.x) {  // CTAs stride over the blocks
  const PadBlock b = P.blocks[bi];
  const double* __restrict__ s = P.src[b.arr] + b.src;
  double* __restrict__ d = P.dst[b.arr] + b.dst;
  // threads over the padded block's elements (consecutive threads: consecutive
  // destination elements), 4 loads in flight per thread before their stores
  if ((int64_t)b.drows * b.dcols >= (1ll << 31)) {  // huge leaf blocks: 64-bit index math
    for (int64_t e = threadIdx.x; e < (int64_t)b.drows * b.dcols; e += kThreads) {
      const int64_t r = e / b.dcols, c = e - r * b.dcols;
      d[e] = (r < b.rows && c < b.cols) ? __ldg(s + r * b.cols + c) : 0.0;
    }
    continue;
  }
  const int tot = b.drows * b.dcols;  // 32-bit index math (a 64-bit division per element was the cost)
  for (int e0 = threadIdx.x; e0 < tot; e0 += 4 * kThreads) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * kThreads;
      const int r = e / b.dcols, c = e - r * b.dcols;
      v[u] = (e < tot && r < b.rows && c < b.cols) ? __ldg(s + r * b.cols + c) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * kThreads;
      if (e < tot) d[e] = v[u];
    }
  }
 }
}

}  // namespace hm
