// hm_fast.cuh — the tuned sm_100a kernels. The generic kernels in
// hm_kernels.cuh remain as the fallback for shapes these do not cover (leaf
// sizes not multiple of 64, ranks that are not 8/16/32/64, ...).
//
// nrhs == 1  (HBM-bound GEMV regime, BASELINE configs 3 (m=1) and 5):
//   vt_gemv_kernel<K>   all levels' V_l^T x in one pass over row tiles;
//   leaf_gemv_kernel<K> per leaf y = D_i x_i + sum_l U_l(I_i) t_l.
//   128-bit streaming loads (ld.global.cs), warp-shuffle reductions,
//   fixed-order cross-warp sums through shared memory.
// nrhs >= 2  (fp64 tensor-core regime, configs 2, 3 (m=8,64), 4):
//   DMMA = mma.sync.aligned.m8n8k4.row.col.f64 (SASS DMMA.8x8x4) — on sm_100a
//   the fp64 tensor path; tcgen05.mma has no f64 kind. Fragments are fed
//   straight from 128-bit global loads, permuting the contraction index so that
//   one LDG.128 feeds two DMMAs (the sum is order-free in exact arithmetic):
//     leaf_mma_kernel       Y_i = [D_i | U_1 | .. | U_S](I_i) . [X_i; T_1; ..; T_S]
//     vt_batched_kernel     t_j = A_j^T B_j for a batch of segments (HSS Step 1
//                           per leaf; HSS upsweep per node with A = W, B = children)
//     vt_mma_levels_kernel  HODLR: every level's V_l^T X over 8-leaf row tiles
//     hss_down_mma_kernel   HSS coupling + downsweep per node:
//                           y_j = S_w x_sib + R_w y_parent
#pragma once
#include <cooperative_groups.h>
#include <cstdint>
#include <cuda_runtime.h>

#include "hm_kernels.cuh"

namespace hm {

// ------------------------------------------------------------ primitives --

// Streaming (evict-first, ld.global.cs) loads for data read exactly once.
__device__ __forceinline__ double2 ldg_stream2(const double* p) {
  double2 v;
  asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ double ldg_stream(const double* p) {
  double v;
  asm volatile("ld.global.cs.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
// Register fence: every value passed must be available here, and nothing that
// uses it may move above. Placed after a batch of (volatile, hence ordered)
// loads it keeps the whole batch in flight before the first use — ptxas would
// otherwise interleave each load with its FMAs to save registers.
__device__ __forceinline__ void reg_fence(double2& v) { asm volatile("" : "+d"(v.x), "+d"(v.y)); }
__device__ __forceinline__ double2 ldg2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }
// Coherent (L2) load for data written earlier in the same launch (cooperative
// kernels): never the non-coherent read-only path.
__device__ __forceinline__ double ldg_cg(const double* p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
template <bool COH>
__device__ __forceinline__ double ld_operand(const double* p) {
  if constexpr (COH) return ldg_cg(p);
  else return __ldg(p);
}

// D (8x8) += A (8x4, row) * B (4x8, col). Lane l holds a = A[l>>2][l&3],
// b = B[l&3][l>>2], c0/c1 = C[l>>2][2(l&3)], C[l>>2][2(l&3)+1].
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) v += __shfl_xor_sync(0xffffffffu, v, w);
  return v;
}

// =================================================================== m == 1 ==

// vt_gemv: one CTA = 8 warps = 8 leaves (tile = 8 b rows); warp w owns the b
// rows of leaf w of the tile. For every level: the warp streams V_l over its
// rows as consecutive 128-bit chunks (64 doubles per warp instruction, i.e.
// 64/K rows), lane l always sees the same rank columns a = (2l) % K, (2l+1) % K,
// so accumulation stays in registers; then a butterfly over the lanes sharing
// a column, and a fixed-order sum over the warps of each node.
struct VtGemvParams {
  const double* X;   // [n]
  int64_t n, b;
  int32_t nlev;
  VtLevel lev[kMaxLevels];  // partial used for levels with s > 8 b
};

template <int K>
__global__ void __launch_bounds__(256) vt_gemv_kernel(const VtGemvParams P) {
  static_assert(K == 1 || K == 2 || K == 4 || K == 8 || K == 16 || K == 32 || K == 64, "K");
  constexpr int kPerChunk = 64;                 // doubles per warp instruction (32 lanes x 2)
  constexpr int kRowsPerChunk = (K >= 64) ? 1 : kPerChunk / K;
  constexpr int kChunksPerRow = (K >= 64) ? K / kPerChunk : 1;
  __shared__ double red[8][K];
  extern __shared__ double xs_all[];  // x of the tile, [8 b]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t b = P.b;
  const int64_t tile = 8 * b;
  const int64_t row0 = (int64_t)blockIdx.x * tile + (int64_t)warp * b;  // this warp's leaf
  for (int64_t e = threadIdx.x; e < tile; e += 256) xs_all[e] = __ldg(P.X + (int64_t)blockIdx.x * tile + e);
  __syncthreads();
  const double* xw = xs_all + (int64_t)warp * b;
  for (int L = 0; L < P.nlev; ++L) {
    const VtLevel lv = P.lev[L];
    const double* V = lv.V + row0 * K;
    const int64_t nchunk = b * K / kPerChunk;    // b % 64 == 0 guaranteed by dispatch
    double acc0 = 0.0, acc1 = 0.0;
    int64_t c = 0;
#pragma unroll 1
    for (; c + 4 <= nchunk; c += 4) {
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = ldg_stream2(V + (c + u) * kPerChunk + 2 * lane);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t e = (c + u) * kPerChunk + 2 * lane;  // element index within the warp's block
        const int64_t r = e / K;
        if (K == 1) {
          const double2 x = *reinterpret_cast<const double2*>(xw + r);
          acc0 = fma(v[u].x, x.x, acc0);
          acc1 = fma(v[u].y, x.y, acc1);
        } else {
          const double x = xw[r];
          acc0 = fma(v[u].x, x, acc0);
          acc1 = fma(v[u].y, x, acc1);
        }
      }
    }
    for (; c < nchunk; ++c) {
      const double2 v = ldg_stream2(V + c * kPerChunk + 2 * lane);
      const int64_t e = c * kPerChunk + 2 * lane;
      const int64_t r = e / K;
      if (K == 1) {
        acc0 = fma(v.x, xw[r], acc0);
        acc1 = fma(v.y, xw[r + 1], acc1);
      } else {
        const double x = xw[r];
        acc0 = fma(v.x, x, acc0);
        acc1 = fma(v.y, x, acc1);
      }
    }
    // lanes sharing rank column: l == l' (mod K/2) (K >= 2); K == 1: everyone
    if (K == 1) {
      double s = warp_sum(acc0 + acc1);
      if (lane == 0) red[warp][0] = s;
    } else if (K < 64) {
#pragma unroll
      for (int w = 16; w >= K / 2 && w >= 1; w >>= 1) {
        acc0 += __shfl_xor_sync(0xffffffffu, acc0, w);
        acc1 += __shfl_xor_sync(0xffffffffu, acc1, w);
      }
      if (lane < K / 2) {
        red[warp][2 * lane] = acc0;
        red[warp][2 * lane + 1] = acc1;
      }
    } else {
      red[warp][2 * lane] = acc0;
      red[warp][2 * lane + 1] = acc1;
    }
    (void)kRowsPerChunk;
    (void)kChunksPerRow;
    __syncthreads();
    // combine warps: node size s (multiple of b): groups of g = min(8, s/b) warps
    const int64_t g = lv.s >= tile ? 8 : lv.s / b;
    const int ngroups = (int)(8 / g);
    for (int o = threadIdx.x; o < ngroups * K; o += 256) {
      const int grp = o / K, a = o - grp * K;
      double s = 0.0;
      for (int w = 0; w < g; ++w) s += red[grp * g + w][a];
      const int64_t rfirst = (int64_t)blockIdx.x * tile + grp * g * b;
      if (lv.s > tile) {
        lv.partial[(int64_t)blockIdx.x * K + a] = s;
      } else {
        lv.out[(rfirst / lv.s) * K + a] = s;
      }
    }
    __syncthreads();
  }
}

// leaf_gemv: one CTA (256 threads) per leaf. D part: warp w owns rows
// w, w+8, ...; a row is b doubles = NCH = b/64 128-bit chunks per lane; ROWS
// rows x NCH chunks (all compile-time) are requested before the first FMA, so
// every warp keeps ROWS*NCH*512 B of D in flight. U part: thread-per-row over
// every segment (K columns each). NCH = 0: runtime b (any multiple of 64).
#ifndef HM_GEMV_ROWS
#define HM_GEMV_ROWS 4
#endif
//
// DT = true (adjoint): the leaf term is D_i^T x_i. The same
// row-major 128-bit stream of D; warp w owns rows w, w+8, ..; lane l keeps the
// partial sums of columns 64c + 2l, 64c + 2l + 1 in registers (x[r] broadcast
// from shared memory); the 8 warps' partials are summed in a fixed order.
//
// VARK = true (per-level ranks on the uniform tree): K is the largest
// rank; segment s has its own rank P.seg[s].k (a power of two <= K).
template <int K, int NCH, int ROWS, bool DT = false, bool VARK = false>
__global__ void __launch_bounds__(256) leaf_gemv_kernel(const LeafParams P) {
  extern __shared__ double sm[];
  const int64_t leaf = blockIdx.x;
  const int64_t b = NCH > 0 ? 64 * NCH : P.b;
  const int64_t r0 = leaf * b;
  double* xs = sm;            // [b]
  double* yd = sm + b;        // [b]
  double* ts = sm + 2 * b;    // [nseg][K]
  double* red = ts + P.nseg * K;  // DT: [8][b] per-warp column partials
  for (int64_t e = threadIdx.x; e < b; e += 256) xs[e] = __ldg(P.X + r0 + e);
  for (int s = 0; s < P.nseg; ++s) {
    const LeafSeg sg = P.seg[s];
    const int64_t node = (leaf >> sg.shift) ^ sg.xr;
    const int kk = VARK ? sg.k : K;
    for (int a = threadIdx.x; a < kk; a += 256) ts[s * K + a] = __ldg(sg.T + node * kk + a);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* Di = P.D + leaf * b * b;
  const int nch = NCH > 0 ? NCH : (int)(b / 64);
  if constexpr (DT) {
    if constexpr (NCH > 0) {
      double2 acc[NCH];
#pragma unroll
      for (int c = 0; c < NCH; ++c) acc[c] = make_double2(0.0, 0.0);
      for (int64_t rb = warp; rb < b; rb += 8 * ROWS) {
        double2 v[ROWS][NCH];
#pragma unroll
        for (int u = 0; u < ROWS; ++u)
#pragma unroll
          for (int c = 0; c < NCH; ++c) v[u][c] = ldg_stream2(Di + (rb + 8 * u) * b + 64 * c + 2 * lane);
#pragma unroll
        for (int u = 0; u < ROWS; ++u)
#pragma unroll
          for (int c = 0; c < NCH; ++c) reg_fence(v[u][c]);
#pragma unroll
        for (int u = 0; u < ROWS; ++u) {
          const double x = xs[rb + 8 * u];
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            acc[c].x = fma(v[u][c].x, x, acc[c].x);
            acc[c].y = fma(v[u][c].y, x, acc[c].y);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < NCH; ++c)
        *reinterpret_cast<double2*>(red + (int64_t)warp * b + 64 * c + 2 * lane) = acc[c];
    } else {
      for (int c = 0; c < nch; ++c) {
        double2 acc = make_double2(0.0, 0.0);
        for (int64_t r = warp; r < b; r += 8) {
          const double2 v = ldg_stream2(Di + r * b + 64 * c + 2 * lane);
          const double x = xs[r];
          acc.x = fma(v.x, x, acc.x);
          acc.y = fma(v.y, x, acc.y);
        }
        *reinterpret_cast<double2*>(red + (int64_t)warp * b + 64 * c + 2 * lane) = acc;
      }
    }
    __syncthreads();
    for (int64_t col = threadIdx.x; col < b; col += 256) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) s += red[(int64_t)w * b + col];
      yd[col] = s;
    }
  }
  for (int64_t rb = warp; !DT && rb < b; rb += 8 * ROWS) {
    double acc[ROWS];
#pragma unroll
    for (int u = 0; u < ROWS; ++u) acc[u] = 0.0;
    if constexpr (NCH > 0) {
      double2 v[ROWS][NCH];
#pragma unroll
      for (int u = 0; u < ROWS; ++u)
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          const int64_t r = rb + 8 * u;  // b = 64 NCH is a multiple of 8 ROWS: always a row
          v[u][c] = ldg_stream2(Di + r * b + 64 * c + 2 * lane);
        }
#pragma unroll
      for (int u = 0; u < ROWS; ++u)
#pragma unroll
        for (int c = 0; c < NCH; ++c) reg_fence(v[u][c]);
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const double2 x = *reinterpret_cast<const double2*>(xs + 64 * c + 2 * lane);
#pragma unroll
        for (int u = 0; u < ROWS; ++u) acc[u] = fma(v[u][c].y, x.y, fma(v[u][c].x, x.x, acc[u]));
      }
    } else {
      for (int c = 0; c < nch; ++c) {
        double2 v[ROWS];
#pragma unroll
        for (int u = 0; u < ROWS; ++u) {
          const int64_t r = rb + 8 * u;
          v[u] = (r < b) ? ldg_stream2(Di + r * b + 64 * c + 2 * lane) : make_double2(0.0, 0.0);
        }
        const double2 x = *reinterpret_cast<const double2*>(xs + 64 * c + 2 * lane);
#pragma unroll
        for (int u = 0; u < ROWS; ++u) acc[u] = fma(v[u].y, x.y, fma(v[u].x, x.x, acc[u]));
      }
    }
#pragma unroll
    for (int u = 0; u < ROWS; ++u) {
      const double s = warp_sum(acc[u]);
      const int64_t r = rb + 8 * u;
      if (lane == 0 && r < b) yd[r] = s;
    }
  }
  // U part, thread per row
  double yu[4];
  int nr = 0;
  for (int64_t r = threadIdx.x; r < b; r += 256, ++nr) {
    double u = 0.0;
    for (int s = 0; s < P.nseg; ++s) {
      const int kk = VARK ? P.seg[s].k : K;
      const double* Ur = P.seg[s].A + (r0 + r) * kk;
      const double* t = ts + s * K;
      if (K == 1 || (VARK && kk == 1)) {
        u = fma(ldg_stream(Ur), t[0], u);
      } else {
#pragma unroll
        for (int a = 0; a < K; a += 2) {
          if (VARK && a >= kk) break;
          const double2 w = ldg_stream2(Ur + a);
          u = fma(w.y, t[a + 1], fma(w.x, t[a], u));
        }
      }
    }
    if (nr < 4) yu[nr] = u;
  }
  __syncthreads();
  nr = 0;
  for (int64_t r = threadIdx.x; r < b; r += 256, ++nr) P.Y[r0 + r] = yd[r] + yu[nr];
}

// ------------------------------------------------ TMA bulk-copy leaf GEMV --
// leaf_gemv_tma: persistent CTAs (one per SM), warp-specialised. One producer
// thread streams every leaf's D rows and U_l rows with 1-D bulk async copies
// (cp.async.bulk, SASS UBLKCP) into an NS-stage shared-memory ring, completion
// signalled on mbarriers (expect_tx); 8 consumer warps compute from shared
// memory and release stages through "empty" mbarriers. Deep, register-free
// memory-level parallelism (NS x 32 KB in flight per SM) for the pure-HBM
// nrhs = 1 leaf pass (BASELINE configs 3 (m=1) and 5).

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// Bounded wait: a protocol bug traps (a reported launch error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  for (uint32_t it = 0; it < (1u << 28); ++it) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
  }
  __trap();
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

constexpr int kTmaChunkBytes = 32 * 1024;
constexpr int kTmaConsumers = 8;  // warps

// Per leaf: nD chunks of `rpc` D rows, then nU chunks of G consecutive U segments.
template <int K, int NCH>
__global__ void __launch_bounds__(32 * (kTmaConsumers + 1), 1)
    leaf_gemv_tma_kernel(const LeafParams P, int64_t nleaves, int NS) {
  constexpr int B = 64 * NCH;
  constexpr int RPC = kTmaChunkBytes / (B * 8);          // D rows per chunk
  constexpr int SEGB = B * K * 8;                        // bytes of one U segment of a leaf
  constexpr int G = SEGB >= kTmaChunkBytes ? 1 : kTmaChunkBytes / SEGB;  // segments per U chunk
  static_assert(RPC >= 1 && RPC % 1 == 0, "leaf too large for a 32 KB chunk row");
  extern __shared__ __align__(128) unsigned char tsm[];
  unsigned char* ring = tsm;
  uint64_t* full = reinterpret_cast<uint64_t*>(tsm + (size_t)NS * kTmaChunkBytes);
  uint64_t* empty = full + NS;
  double* xs = reinterpret_cast<double*>(empty + NS);  // [B]
  double* yd = xs + B;                                 // [B]
  double* ts = yd + B;                                 // [nseg][K]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nseg = P.nseg;
  const int nD = B / RPC;
  const int nU = (nseg + G - 1) / G;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kTmaConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kTmaConsumers) {
    // ---------------- producer (one thread) ----------------
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int64_t leaf = blockIdx.x; leaf < nleaves; leaf += gridDim.x) {
        const unsigned char* Dl = reinterpret_cast<const unsigned char*>(P.D + leaf * B * B);
        for (int c = 0; c < nD; ++c) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], RPC * B * 8);
          bulk_g2s(ring + (size_t)s * kTmaChunkBytes, Dl + (size_t)c * RPC * B * 8, RPC * B * 8, &full[s]);
          if (++s == NS) { s = 0; ph ^= 1; }
        }
        for (int g = 0; g < nU; ++g) {
          const int s0 = g * G, s1 = min(nseg, s0 + G);
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], (uint32_t)(s1 - s0) * SEGB);
          for (int sg = s0; sg < s1; ++sg)
            bulk_g2s(ring + (size_t)s * kTmaChunkBytes + (size_t)(sg - s0) * SEGB, P.seg[sg].A + leaf * B * K, SEGB,
                     &full[s]);
          if (++s == NS) { s = 0; ph ^= 1; }
        }
      }
    }
    return;
  }
  // ---------------- consumers (8 warps, 256 threads) ----------------
  int s = 0;
  uint32_t ph = 0;
  const int t = threadIdx.x;
  for (int64_t leaf = blockIdx.x; leaf < nleaves; leaf += gridDim.x) {
    const int64_t r0 = leaf * B;
    named_bar(1, 32 * kTmaConsumers);  // previous leaf fully written out
    for (int e = t; e < B; e += 32 * kTmaConsumers) xs[e] = __ldg(P.X + r0 + e);
    for (int sg = 0; sg < nseg; ++sg) {
      const LeafSeg g = P.seg[sg];
      const int64_t node = (leaf >> g.shift) ^ g.xr;
      for (int a = t; a < K; a += 32 * kTmaConsumers) ts[sg * K + a] = __ldg(g.T + node * K + a);
    }
    named_bar(1, 32 * kTmaConsumers);
    double2 xr[NCH];
#pragma unroll
    for (int j = 0; j < NCH; ++j) xr[j] = *reinterpret_cast<const double2*>(xs + 64 * j + 2 * lane);
    for (int c = 0; c < nD; ++c) {
      mbar_wait(&full[s], ph);
      const double* chunk = reinterpret_cast<const double*>(ring + (size_t)s * kTmaChunkBytes);
      for (int rr = warp; rr < RPC; rr += kTmaConsumers) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          const double2 v = *reinterpret_cast<const double2*>(chunk + rr * B + 64 * j + 2 * lane);
          acc = fma(v.y, xr[j].y, fma(v.x, xr[j].x, acc));
        }
        acc = warp_sum(acc);
        if (lane == 0) yd[c * RPC + rr] = acc;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == NS) { s = 0; ph ^= 1; }
    }
    // U segments: thread per row (rows t, t + 256, ...)
    double yu[(B + 255) / 256];
#pragma unroll
    for (int i = 0; i < (B + 255) / 256; ++i) yu[i] = 0.0;
    for (int g = 0; g < nU; ++g) {
      mbar_wait(&full[s], ph);
      const double* chunk = reinterpret_cast<const double*>(ring + (size_t)s * kTmaChunkBytes);
      const int s0 = g * G, s1 = min(nseg, s0 + G);
      for (int sg = s0; sg < s1; ++sg) {
        const double* Us = chunk + (size_t)(sg - s0) * B * K;
        const double* tv = ts + sg * K;
#pragma unroll
        for (int i = 0; i < (B + 255) / 256; ++i) {
          const int r = t + 256 * i;
          if (r < B) {
            double u = 0.0;
#pragma unroll
            for (int a = 0; a < K; ++a) u = fma(Us[r * K + ((a + r) & (K - 1))], tv[(a + r) & (K - 1)], u);
            yu[i] += u;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == NS) { s = 0; ph ^= 1; }
    }
    named_bar(1, 32 * kTmaConsumers);  // every yd row written
#pragma unroll
    for (int i = 0; i < (B + 255) / 256; ++i) {
      const int r = t + 256 * i;
      if (r < B) P.Y[r0 + r] = yd[r] + yu[i];
    }
  }
}

// =================================================================== m >= 2 ==

#ifndef HM_RM_PF
#define HM_RM_PF 2
#endif
// Tuning: the DMMA kernels take MINB (minimum resident CTAs per SM for the
// launch bounds; 0 = unconstrained) and the A-stream prefetch depth PF as
// template parameters; the host picks them per shape (hm_leaf.cu, measured on
// B200: profiles/r01_tuning.md).

// cp.async (LDGSTS) 16-byte global -> shared copies: the whole staging of a
// block is in flight at once, with no register round trip.
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Stage `rows` x `cols` doubles (global, row stride lds) into shared memory
// rows of stride zs, zero-filling columns cols .. mp-1. All threads of the CTA
// take part; the caller issues cp_async_wait_all() + __syncthreads(). cp.async.cg
// reads through L2, so this is also coherent inside a cooperative kernel.
__device__ __forceinline__ void stage_rows_async(double* dst, int zs, const double* src, int64_t lds, int rows,
                                                 int cols, int mp) {
  const bool vec = ((cols & 1) == 0) && ((lds & 1) == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0) &&
                   ((zs & 1) == 0) && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
  if (vec) {
    const int h = cols >> 1;  // 16-byte chunks per row
    for (int e = threadIdx.x; e < rows * h; e += blockDim.x) {
      const int r = e / h, c = (e - r * h) * 2;
      cp_async16(dst + r * zs + c, src + (int64_t)r * lds + c);
    }
  } else {
    for (int e = threadIdx.x; e < rows * cols; e += blockDim.x) {
      const int r = e / cols, c = e - r * cols;
      dst[r * zs + c] = ldg_cg(src + (int64_t)r * lds + c);
    }
  }
  if (mp > cols)
    for (int e = threadIdx.x; e < rows * (mp - cols); e += blockDim.x) {
      const int r = e / (mp - cols), c = cols + (e - r * (mp - cols));
      dst[r * zs + c] = 0.0;
    }
}

// One warp accumulates C (8 RG rows x 8 NT cols) += E (rows, K) . Z (K, cols)
// where E rows are row-major in global memory (lda) and Z (row stride zs) is
// in shared memory (ZG = false, zero-padded columns) or global memory (ZG =
// true, columns >= zvalid read as 0). K % 8 == 0. One LDG.128 per row group
// and 8 k-indices feeds two DMMAs: k = kc+2j (".x") and kc+2j+1 (".y"),
// j = lane & 3 — a permutation of the contraction index. The A stream is
// software-pipelined: groups of PF k-chunks ping-pong between two register
// buffers, so the next group's loads are in flight while the current one
// feeds the tensor pipe.
template <int RG, int NT, bool ZG, bool COH, int PF>
__device__ __forceinline__ void rm_group(double (&acc)[RG][NT][2], const double2 (&a)[PF][RG], const double* Z,
                                         int64_t zs, int q, int nq, const bool (&colok)[NT], int lane) {
  const int j = lane & 3, i = lane >> 2;
#pragma unroll
  for (int u = 0; u < PF; ++u) {
    if (q + u >= nq) break;  // warp-uniform
    const double* zr = Z + (int64_t)(8 * (q + u) + 2 * j) * zs + i;
    double b0[NT], b1[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      b0[nt] = colok[nt] ? (ZG ? ld_operand<COH>(zr + nt * 8) : zr[nt * 8]) : 0.0;
      b1[nt] = colok[nt] ? (ZG ? ld_operand<COH>(zr + zs + nt * 8) : zr[zs + nt * 8]) : 0.0;
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int rg = 0; rg < RG; ++rg) dmma(acc[rg][nt][0], acc[rg][nt][1], a[u][rg].x, b0[nt]);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int rg = 0; rg < RG; ++rg) dmma(acc[rg][nt][0], acc[rg][nt][1], a[u][rg].y, b1[nt]);
  }
}

// Row of the warp's tile rg held by lane group i (= lane >> 2): 8 rg + i, or,
// with PAIR (the row order of warp_dt_mma, adjoint leaf pass), tiles 2pr and
// 2pr+1 interleaved over 16 rows: 16 pr + 2 i + (rg & 1).
template <bool PAIR>
__device__ __forceinline__ int tile_row(int rg, int i) {
  return PAIR ? 16 * (rg >> 1) + 2 * i + (rg & 1) : 8 * rg + i;
}

// Load policy of the row-major A stream (leaf pass D and U rows): a warp
// instruction covers 64 B of 8 rows, so every 128-B line is completed by a
// later instruction. 0: ld.global.cs (evict-first); 1: ld.global.nc (evict
// normal); 2: evict-normal with an L2 256-B prefetch of the line pair.
#ifndef HM_LDA_POLICY
#define HM_LDA_POLICY 2  // measured: config-4 leaf DRAM read 7.60 -> 6.71 GB (= algorithmic), 1539 -> 1485 us
#endif
__device__ __forceinline__ double2 ld_a_stream2(const double* p) {
#if HM_LDA_POLICY == 0
  return ldg_stream2(p);
#elif HM_LDA_POLICY == 1
  return __ldg(reinterpret_cast<const double2*>(p));
#else
  double2 v;
  asm volatile("ld.global.nc.L2::256B.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
#endif
}

template <int RG, int PF, bool PAIR = false>
__device__ __forceinline__ void rm_load(double2 (&a)[PF][RG], const double* base, int64_t lda, int q, int nq) {
#pragma unroll
  for (int u = 0; u < PF; ++u)
#pragma unroll
    for (int rg = 0; rg < RG; ++rg)
      a[u][rg] = (q + u < nq) ? ld_a_stream2(base + (int64_t)tile_row<PAIR>(rg, 0) * lda + 8 * (q + u))
                              : make_double2(0.0, 0.0);
}

template <int RG, int NT, bool ZG, bool COH = false, int PF = HM_RM_PF, bool PAIR = false>
__device__ __forceinline__ void warp_rowmajor_mma(double (&acc)[RG][NT][2], const double* __restrict__ E, int64_t lda,
                                                  int K, const double* Z, int64_t zs, int zvalid, int lane) {
  const int j = lane & 3, i = lane >> 2;
  const double* base = E + (int64_t)(PAIR ? 2 * i : i) * lda + 2 * j;
  bool colok[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) colok[nt] = !ZG || (nt * 8 + i) < zvalid;
  const int nq = K / 8;
  double2 a0[PF][RG], a1[PF][RG];
  rm_load<RG, PF, PAIR>(a0, base, lda, 0, nq);
  for (int q = 0; q < nq; q += 2 * PF) {
    rm_load<RG, PF, PAIR>(a1, base, lda, q + PF, nq);
    rm_group<RG, NT, ZG, COH, PF>(acc, a0, Z, zs, q, nq, colok, lane);
    if (q + PF >= nq) break;
    rm_load<RG, PF, PAIR>(a0, base, lda, q + 2 * PF, nq);
    rm_group<RG, NT, ZG, COH, PF>(acc, a1, Z, zs, q + PF, nq, colok, lane);
  }
}

// Adjoint leaf term: one warp accumulates C += D^T(rows, :) Z
// for its 8 RG output rows, D [K][ldd] row-major in global memory (Dc points at
// the warp's first column). A fragment of tile rg: D[k][tile_row(rg, i)] with
// k = 4q + (lane & 3). For even RG one LDG.128 of two adjacent columns feeds
// the two interleaved tiles of a pair (PAIR row order); for RG = 1 a 64-bit
// load per fragment. B fragments: rows 4q + (lane & 3) of Z (shared memory).
template <int RG, int NT>
__device__ __forceinline__ void warp_dt_mma(double (&acc)[RG][NT][2], const double* __restrict__ Dc, int64_t ldd, int K,
                                            const double* Z, int64_t zs, int lane) {
  constexpr bool PAIR = (RG % 2 == 0);
  constexpr int PF = 4;  // k-steps (4 rows of D each) per batch of loads
  const int j = lane & 3, i = lane >> 2;
  const double* ap = Dc + (int64_t)j * ldd + (PAIR ? 2 * i : i);
  const double* zp = Z + (int64_t)j * zs + i;
#pragma unroll 1
  for (int q = 0; q < K / 4; q += PF) {  // K % 16 == 0 (leaf sizes 64, 128, 256)
    double a[PF][RG];
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const double* ar = ap + (int64_t)(q + u) * 4 * ldd;
      if constexpr (PAIR) {
#pragma unroll
        for (int pr = 0; pr < RG / 2; ++pr) {
          const double2 v = ldg_stream2(ar + 16 * pr);
          a[u][2 * pr] = v.x;
          a[u][2 * pr + 1] = v.y;
        }
      } else {
#pragma unroll
        for (int rg = 0; rg < RG; ++rg) a[u][rg] = ldg_stream(ar + 8 * rg);
      }
    }
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      double bf[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) bf[nt] = zp[(int64_t)(q + u) * 4 * zs + nt * 8];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int rg = 0; rg < RG; ++rg) dmma(acc[rg][nt][0], acc[rg][nt][1], a[u][rg], bf[nt]);
    }
  }
}

// leaf_mma: grid (chunks of NT*8 columns, leaves); 8 warps; warp w owns rows
// [w*8*RG, (w+1)*8*RG) of the leaf (b = 64 RG). Z = [X_i; T_1; ..; T_S] staged
// in shared memory with row stride NT*8+4 (conflict-free B fragments).
// DT (adjoint): the leaf term is D_i^T X_i (warp_dt_mma); for even RG the
// warp's rows are in PAIR order, which the U segments and the store follow.

template <int RG, int NT, int PF, int MINB, bool DT = false>
__global__ void __launch_bounds__(256, MINB) leaf_mma_kernel(const LeafParams P) {
  constexpr bool PAIR = DT && (RG % 2 == 0);
  extern __shared__ double sm[];
  constexpr int MC = NT * 8;
  // Row strides of the staged operand (conflict-free 64-bit fragment loads, see
  // hm_tree.cuh): rows 2j apart (row-major pattern) need ZS = 2 (mod 4); the
  // adjoint's D^T pattern reads the X rows j apart and needs 4 (mod 8).
  constexpr int ZS = MC + 2;
  constexpr int ZSX = DT ? MC + 4 : ZS;  // X region
  const int nchunks = (P.m + MC - 1) / MC;
  const int64_t leaf = blockIdx.x / nchunks;
  const int c0 = (int)(blockIdx.x - leaf * nchunks) * MC;
  const int64_t b = P.b;  // == 64 * RG
  const int64_t r0 = leaf * b;
  const int m = P.m;
  double* Z = sm;
  const int mc = min(MC, m - c0);
  stage_rows_async(Z, ZSX, P.X + r0 * m + c0, m, (int)b, mc, MC);
  double* ZT = Z + b * ZSX;  // T region
  int64_t zoff = 0;
  for (int s = 0; s < P.nseg; ++s) {
    const LeafSeg sg = P.seg[s];
    const int64_t node = (leaf >> sg.shift) ^ sg.xr;
    stage_rows_async(ZT + zoff * ZS, ZS, sg.T + node * sg.k * m + c0, m, sg.k, mc, MC);
    zoff += sg.k;
  }
  cp_async_wait_all();
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc[RG][NT][2];
#pragma unroll
  for (int rg = 0; rg < RG; ++rg)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[rg][nt][0] = acc[rg][nt][1] = 0.0;
  const int64_t wrow = (int64_t)warp * 8 * RG;
  if constexpr (DT) warp_dt_mma<RG, NT>(acc, P.D + leaf * b * b + wrow, b, (int)b, Z, ZSX, lane);
  else warp_rowmajor_mma<RG, NT, false, false, PF>(acc, P.D + leaf * b * b + wrow * b, b, (int)b, Z, ZS, MC, lane);
  zoff = 0;
  for (int s = 0; s < P.nseg; ++s) {
    const LeafSeg sg = P.seg[s];
    warp_rowmajor_mma<RG, NT, false, false, PF, PAIR>(acc, sg.A + (r0 + wrow) * sg.k, sg.k, sg.k, ZT + zoff * ZS,
                                                      ZS, MC, lane);
    zoff += sg.k;
  }
  const int i = lane >> 2, j = lane & 3;
#pragma unroll
  for (int rg = 0; rg < RG; ++rg) {
    double* y = P.Y + (r0 + wrow + tile_row<PAIR>(rg, i)) * m;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int c = c0 + nt * 8 + 2 * j;
      if (c + 1 < m) {
        if ((m & 1) == 0) {
          *reinterpret_cast<double2*>(y + c) = make_double2(acc[rg][nt][0], acc[rg][nt][1]);
        } else {
          y[c] = acc[rg][nt][0];
          y[c + 1] = acc[rg][nt][1];
        }
      } else if (c < m) {
        y[c] = acc[rg][nt][0];
      }
    }
  }
}

// HSS Step 4 with the leaf level's coupling + downsweep folded in (Fig. 5
// right): per leaf i = 2q + w the CTA first forms
//   y_i = S_w x_{i^1} + R_{p-1,q}[w] y_{p-1,q}        (KT x MC columns c0..)
// — S_w, R rows as A fragments from global memory, x_{i^1} and y_{p-1,q}
// staged with X(I_i) — keeps it in shared memory in place of the y_i the
// separate downsweep launch would have written, then runs the leaf pass
// Y(I_i) = D_i X(I_i) + U_i y_i of leaf_mma_kernel. Saves the level-p y blocks'
// write and re-read (and one launch). Forward product, p >= 2, one U segment.
struct LeafDownParams {
  const double* B;    // cores, pair (l, q) at 2^l - 1 + q ([2][KT][KT])
  const double* R;    // translations, node (l, i) at 2^l - 2 + i ([2KT][KT])
  const double* xh;   // x of the leaves: leaf i at i KT m
  const double* yhp;  // y of level p-1: node q at q KT m
  int32_t p;
  int32_t pad;
};

template <int RG, int NT, int PF, int MINB, int KT>
__global__ void __launch_bounds__(256, MINB) leaf_mma_down_kernel(const LeafParams P, const LeafDownParams Q) {
  extern __shared__ double sm[];
  constexpr int MC = NT * 8, ZS = MC + 2;
  const int nchunks = (P.m + MC - 1) / MC;
  const int64_t leaf = blockIdx.x / nchunks;
  const int c0 = (int)(blockIdx.x - leaf * nchunks) * MC;
  const int64_t b = P.b;  // == 64 RG
  const int64_t r0 = leaf * b;
  const int m = P.m;
  const int mc = min(MC, m - c0);
  const int64_t km = (int64_t)KT * m;
  const int64_t q = leaf >> 1;
  const int w = (int)(leaf & 1);
  double* Z = sm;                 // X(I_i): b rows
  double* ZT = Z + b * ZS;        // x_{i^1} (KT rows), then y_i (KT rows)
  double* ZP = ZT + KT * ZS;      // y_{p-1,q}: KT rows
  stage_rows_async(Z, ZS, P.X + r0 * m + c0, m, (int)b, mc, MC);
  stage_rows_async(ZT, ZS, Q.xh + (leaf ^ 1) * km + c0, m, KT, mc, MC);
  stage_rows_async(ZP, ZS, Q.yhp + q * km + c0, m, KT, mc, MC);
  cp_async_wait_all();
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = lane >> 2, j = lane & 3;
  // y_i: (KT / 8) x NT tiles of 8 x 8, over the 8 warps; K = KT from each operand
  constexpr int TILES = (KT / 8) * NT, TPW = (TILES + 7) / 8;
  const double* S = Q.B + ((((int64_t)1 << (Q.p - 1)) - 1 + q) * 2 + w) * KT * KT;
  const double* Rw = Q.R + ((((int64_t)1 << (Q.p - 1)) - 2 + q) * 2 * KT + (int64_t)w * KT) * KT;
  double yacc[TPW][1][1][2];
#pragma unroll
  for (int u = 0; u < TPW; ++u) {
    yacc[u][0][0][0] = yacc[u][0][0][1] = 0.0;
    const int t = warp + 8 * u;
    if (t < TILES) {
      const int rt = t % (KT / 8), ct = t / (KT / 8);
      warp_rowmajor_mma<1, 1, false, false, 2>(yacc[u], S + (int64_t)8 * rt * KT, KT, KT, ZT + ct * 8, ZS, MC, lane);
      warp_rowmajor_mma<1, 1, false, false, 2>(yacc[u], Rw + (int64_t)8 * rt * KT, KT, KT, ZP + ct * 8, ZS, MC, lane);
    }
  }
  __syncthreads();  // every warp has read x_{i^1}: its rows now take y_i
#pragma unroll
  for (int u = 0; u < TPW; ++u) {
    const int t = warp + 8 * u;
    if (t < TILES) {
      const int rt = t % (KT / 8), ct = t / (KT / 8);
      double* o = ZT + (8 * rt + i) * ZS + ct * 8 + 2 * j;
      o[0] = yacc[u][0][0][0];
      o[1] = yacc[u][0][0][1];
    }
  }
  __syncthreads();
  double acc[RG][NT][2];
#pragma unroll
  for (int rg = 0; rg < RG; ++rg)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[rg][nt][0] = acc[rg][nt][1] = 0.0;
  const int64_t wrow = (int64_t)warp * 8 * RG;
  warp_rowmajor_mma<RG, NT, false, false, PF>(acc, P.D + leaf * b * b + wrow * b, b, (int)b, Z, ZS, MC, lane);
  warp_rowmajor_mma<RG, NT, false, false, PF>(acc, P.seg[0].A + (r0 + wrow) * KT, KT, KT, ZT, ZS, MC, lane);
#pragma unroll
  for (int rg = 0; rg < RG; ++rg) {
    double* y = P.Y + (r0 + wrow + 8 * rg + i) * m;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int c = c0 + nt * 8 + 2 * j;
      if (c + 1 < m) {
        if ((m & 1) == 0) {
          *reinterpret_cast<double2*>(y + c) = make_double2(acc[rg][nt][0], acc[rg][nt][1]);
        } else {
          y[c] = acc[rg][nt][0];
          y[c + 1] = acc[rg][nt][1];
        }
      } else if (c < m) {
        y[c] = acc[rg][nt][0];
      }
    }
  }
}

// One warp accumulates C (16 MPW x 8 NT) += A^T B over K rows, A [K][lda]
// row-major (the warp's rank columns start at A), B [K][ldb] (columns c0..).
// The 4 rows of one k-step are rows r + (lane & 3). One LDG.128 of A covers 16
// rank columns: ".x" feeds the tile of even columns, ".y" the tile of odd
// columns (output rows permuted back at the store). K % 4 == 0.
template <int MPW, int NT, bool COH = false, int PF = (NT > 4 ? 2 : 4)>
__device__ __forceinline__ void warp_transposed_mma(double (&acc)[2 * MPW][NT][2], const double* __restrict__ A,
                                                    int64_t lda, const double* __restrict__ B, int64_t ldb, int c0,
                                                    int m, int K, int lane) {
  const int j = lane & 3, i = lane >> 2;
  const double* ap = A + (int64_t)j * lda + 2 * i;
  const double* bp = B + (int64_t)j * ldb + c0 + i;
  bool colok[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) colok[nt] = (c0 + nt * 8 + i) < m;
  int q = 0;
#pragma unroll 1
  for (; q + PF <= K / 4; q += PF) {
    double2 a[PF][MPW];
    double bf[PF][NT];
#pragma unroll
    for (int u = 0; u < PF; ++u) {
#pragma unroll
      for (int mp = 0; mp < MPW; ++mp) a[u][mp] = ldg_stream2(ap + (int64_t)(q + u) * 4 * lda + mp * 16);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) bf[u][nt] = colok[nt] ? ld_operand<COH>(bp + (int64_t)(q + u) * 4 * ldb + nt * 8) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < PF; ++u)
#pragma unroll
      for (int mp = 0; mp < MPW; ++mp)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          dmma(acc[2 * mp][nt][0], acc[2 * mp][nt][1], a[u][mp].x, bf[u][nt]);
          dmma(acc[2 * mp + 1][nt][0], acc[2 * mp + 1][nt][1], a[u][mp].y, bf[u][nt]);
        }
  }
  for (; q < K / 4; ++q) {
    double2 a[MPW];
    double bf[NT];
#pragma unroll
    for (int mp = 0; mp < MPW; ++mp) a[mp] = ldg_stream2(ap + (int64_t)q * 4 * lda + mp * 16);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) bf[nt] = colok[nt] ? ld_operand<COH>(bp + (int64_t)q * 4 * ldb + nt * 8) : 0.0;
#pragma unroll
    for (int mp = 0; mp < MPW; ++mp)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        dmma(acc[2 * mp][nt][0], acc[2 * mp][nt][1], a[mp].x, bf[nt]);
        dmma(acc[2 * mp + 1][nt][0], acc[2 * mp + 1][nt][1], a[mp].y, bf[nt]);
      }
  }
}

// Store a warp's (16 MPW) x 8NT result: tile t = 2 mp + e holds rank columns
// a = 16 mp + 2 i + e (i = lane >> 2) relative to the warp's first column;
// columns c0 + 8 nt + 2 (lane&3) + {0,1}, written at (c - cbase).
template <int MPW, int NT>
__device__ __forceinline__ void store_transposed(const double (&acc)[2 * MPW][NT][2], double* out, int64_t ldo, int c0,
                                                 int m, int lane, int cbase = 0) {
  const int i = lane >> 2, j = lane & 3;
#pragma unroll
  for (int t = 0; t < 2 * MPW; ++t) {
    const int a = 16 * (t >> 1) + 2 * i + (t & 1);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int c = c0 + nt * 8 + 2 * j;
      double* o = out + (int64_t)a * ldo + (c - cbase);
      if (c + 1 < m) {
        o[0] = acc[t][nt][0];
        o[1] = acc[t][nt][1];
      } else if (c < m) {
        o[0] = acc[t][nt][0];
      }
    }
  }
}

// Batched t_j = A_j^T B_j ([K][KT])^T [K][m]. Each segment is split over
// (KT/16/MPW) rank-column groups x ceil(m / 8NT) column chunks, one warp each.
struct BatchedVtParams {
  const double* A;  int64_t a_stride;   // A_j = A + j * a_stride, [K][KT]
  const double* B;  int64_t b_stride;   // B_j = B + j * b_stride, [K][m]
  double* out;      int64_t o_stride;   // out_j = out + j * o_stride, [KT][m]
  int64_t count;
  int32_t K, m;
};

// One warp task of the batched product: segment jseg, rank-column group mg,
// column chunk ck.
// k-steps per batch of A/B loads: measured on config 4 Step 1 (r01_tuning.md):
// MPW 1: PF 4 483 us, PF 2 452 us, PF 1 742 us; MPW 2 (one warp, 32 rank
// columns): PF 1 398 us, PF 2 721 us.
template <int KT, int MPW, int NT, bool COH = false, int PF = (NT > 4 ? 2 : (MPW >= 2 ? 1 : 2))>
__device__ __forceinline__ void vt_batched_task(const BatchedVtParams& P, int64_t jseg, int mg, int ck, int lane) {
  const int c0 = ck * NT * 8;
  double acc[2 * MPW][NT][2];
#pragma unroll
  for (int t = 0; t < 2 * MPW; ++t)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[t][nt][0] = acc[t][nt][1] = 0.0;
  warp_transposed_mma<MPW, NT, COH, PF>(acc, P.A + jseg * P.a_stride + mg * 16 * MPW, KT, P.B + jseg * P.b_stride,
                                        P.m, c0, P.m, P.K, lane);
  store_transposed<MPW, NT>(acc, P.out + jseg * P.o_stride + (int64_t)mg * 16 * MPW * P.m, P.m, c0, P.m, lane);
}

template <int KT, int MPW, int NT>
__global__ void __launch_bounds__(256) vt_batched_kernel(const BatchedVtParams P) {
  constexpr int MG = KT / 16 / MPW;  // rank-column groups
  const int lane = threadIdx.x & 31;
  const int nck = (P.m + NT * 8 - 1) / (NT * 8);
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t per = (int64_t)MG * nck;
  const int64_t jseg = gw / per;
  if (jseg >= P.count) return;
  const int sub = (int)(gw - jseg * per);
  vt_batched_task<KT, MPW, NT>(P, jseg, sub % MG, sub / MG, lane);
}

#ifndef HM_VTM_PF
#define HM_VTM_PF(NT) ((NT) > 4 ? 2 : 4)
#endif

// Small ranks (KT = 1, 2, 4, 8; per-level ranks below 16): C (8 x 8NT)
// += A^T B with A [K][KT]. One DMMA tile holds every rank column (rows a < KT
// valid). A k-step's A fragment is A[4q + j][i] (i = lane >> 2, j = lane & 3):
// 4 consecutive rows of KT doubles, one coalesced 64-bit load per lane; B
// fragments X[4q + j][c0 + 8nt + i] straight from global memory.
template <int KT, int NT, int PF>
__device__ __forceinline__ void warp_transposed_mma_small(double (&acc)[1][NT][2], const double* __restrict__ A,
                                                          const double* __restrict__ B, int64_t ldb, int c0, int m,
                                                          int K, int lane) {
  const int j = lane & 3, i = lane >> 2;
  const bool aok = i < KT;
  const double* ap = A + (int64_t)j * KT + (aok ? i : 0);
  const double* bp = B + (int64_t)j * ldb + c0 + i;
  bool colok[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) colok[nt] = (c0 + nt * 8 + i) < m;
  int q = 0;
#pragma unroll 1
  for (; q + PF <= K / 4; q += PF) {
    double a[PF], bf[PF][NT];
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      a[u] = aok ? ldg_stream(ap + (int64_t)(q + u) * 4 * KT) : 0.0;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) bf[u][nt] = colok[nt] ? __ldg(bp + (int64_t)(q + u) * 4 * ldb + nt * 8) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < PF; ++u)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) dmma(acc[0][nt][0], acc[0][nt][1], a[u], bf[u][nt]);
  }
  for (; q < K / 4; ++q) {
    const double a = aok ? ldg_stream(ap + (int64_t)q * 4 * KT) : 0.0;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const double bf = colok[nt] ? __ldg(bp + (int64_t)q * 4 * ldb + nt * 8) : 0.0;
      dmma(acc[0][nt][0], acc[0][nt][1], a, bf);
    }
  }
}
// HODLR, many right-hand sides (m > 16): vt_mma_levels re-reads a tile's X rows
// once per level, and with m = 64 the live X tiles of all resident CTAs (1 MB
// each) exceed L2 — ncu on config 3, m = 64: 8.0 GB of DRAM reads for 2.1 GB of
// V and X. vt_lv_kernel reads X and V exactly once: the CTA walks its 8-leaf
// tile in chunks of R rows; a cp.async pipeline of NS stages holds, per chunk,
// the R rows of X (row stride m_pad + 4) and of every level's V (row stride
// KT + 4); warps own work items (level, 16-rank-column group, column chunk of
// 8 NT) — up to IPW each for NW warps, accumulators in registers across the
// chunks of a node — with A fragments (V, 128-bit) and B fragments (X, 64-bit)
// both from shared memory. NW = 16 warps, NT = 2: with 8 warps and NT = 4
// (ncu, config 3 m = 64) the tensor pipe was 57% active, stalled on DMMA
// dependency waits with 2 warps per SMSP. A node's sum is written when its last chunk is done (nodes
// inside the tile) or as the tile's partial (nodes spanning tiles; fixed-order
// reduce_partials). Shared-memory strides: 128-bit loads of V rows 4q + j,
// columns 2i (8 lanes per wavefront) need KT + 4 = 4 (mod 16) doubles... for
// KT = 16 that is 20; the X rows j apart need m_pad + 4 = 4 (mod 8).
__device__ __forceinline__ void cp_async_commit_group() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_groups() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__host__ __device__ constexpr int vt_lv_vstride(int kt) { return kt + 4; }
__host__ __device__ constexpr int vt_lv_xstride(int mpad) { return mpad + 4; }
// doubles of one pipeline stage: R rows of every level's V and of X
__host__ __device__ constexpr int64_t vt_lv_stage_doubles(int r, int kt, int nlev, int mpad) {
  return (int64_t)r * ((int64_t)nlev * vt_lv_vstride(kt) + vt_lv_xstride(mpad));
}

template <int KT, int NT, int IPW, int R, int NS, int NW>
__global__ void __launch_bounds__(NW * 32, 1) vt_lv_kernel(const VtParams P, int64_t b) {
  extern __shared__ double stg[];
  constexpr int BS = NW * 32;
  constexpr int MC = NT * 8;
  constexpr int G = KT / 16;  // 16-rank-column groups per level
  constexpr int VS = vt_lv_vstride(KT);
  constexpr int VH = KT / 2;  // 16-byte pieces per V row
  constexpr int VP = R * VH;  // pieces per level and chunk
  static_assert(BS % VP == 0 || VP % BS == 0, "V staging split");
  const int m = P.m, nlev = P.nlev;
  const int mp = (m + MC - 1) / MC * MC;
  const int XS = vt_lv_xstride(mp);
  const int sd = (int)vt_lv_stage_doubles(R, KT, nlev, mp);
  const int64_t T = P.tile;  // tile rows: 8 or 4 leaves (the plan's wave balance)
  const int64_t row0 = (int64_t)blockIdx.x * T;
  const int nch = (int)(T / R);
  const int nck = mp / MC;
  const int nitems = nlev * G * nck;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = lane >> 2, j = lane & 3;
  const int xoff = nlev * R * VS;  // X region of a stage

  // staging: per-thread piece coordinates computed once (no division per chunk)
  const int vL0 = BS >= VP ? threadIdx.x / VP : 0, vLs = BS >= VP ? BS / VP : 1;
  const int ve = BS >= VP ? threadIdx.x % VP : threadIdx.x;
  const bool xvec = (m & 1) == 0;
  const int XH = xvec ? m / 2 : m;  // pieces per X row
  const int xr0 = threadIdx.x / XH, xc0 = threadIdx.x % XH, xdr = BS / XH, xdc = BS % XH;
  auto stage = [&](int c) {
    double* dst = stg + (c % NS) * sd;
    const int64_t r0 = row0 + (int64_t)c * R;
    for (int L = vL0; L < nlev; L += vLs) {
      const double* src = P.lev[L].V + r0 * KT;
      double* d = dst + L * R * VS;
      for (int e = ve; e < VP; e += (BS >= VP ? VP : BS)) {
        const int r = e / VH, c2 = (e % VH) * 2;  // VH constexpr: shifts
        cp_async16(d + r * VS + c2, src + r * KT + c2);
      }
    }
    double* dx = dst + xoff;
    const double* xsrc = P.X + r0 * m;
    for (int r = xr0, cc = xc0; r < R;) {
      if (xvec) cp_async16(dx + r * XS + 2 * cc, xsrc + (int64_t)r * m + 2 * cc);
      else dx[r * XS + cc] = __ldg(xsrc + (int64_t)r * m + cc);
      r += xdr;
      cc += xdc;
      if (cc >= XH) { cc -= XH; ++r; }
    }
    cp_async_commit_group();
  };
  // zero the padded X columns of every buffer once (never written by the stages)
  if (mp > m)
    for (int bf = 0; bf < NS; ++bf) {
      double* dx = stg + bf * sd + xoff;
      for (int e = threadIdx.x; e < R * (mp - m); e += BS) {
        const int r = e / (mp - m);
        dx[r * XS + m + (e - r * (mp - m))] = 0.0;
      }
    }

  // work items of this warp, decoded once
  int ia[IPW], ib[IPW], icpn[IPW], icmax[IPW];  // A / B offsets in a stage, chunks per node (0: spans tiles), column limit
  double* iout[IPW];
#pragma unroll
  for (int u = 0; u < IPW; ++u) {
    const int t = warp + NW * u;
    const int tt = t < nitems ? t : 0;
    const int L = tt / (G * nck), rem = tt - L * G * nck;
    const int g = rem / nck, ck = rem - g * nck;
    ia[u] = L * R * VS + j * VS + g * 16 + 2 * i;
    ib[u] = xoff + j * XS + ck * MC + i;
    const VtLevel& lv = P.lev[L];
    const bool inside = lv.s <= T;
    icpn[u] = inside ? (int)(lv.s / R) : 0;
    icmax[u] = m - 2 * j - ck * MC;  // columns ck MC + 8 nt + 2 j (+1) valid while < m
    // node output base (inside: node of the tile's first row; advanced per node) or tile partial
    iout[u] = (inside ? lv.out + (row0 / lv.s) * KT * m : lv.partial + (int64_t)blockIdx.x * KT * m) +
              (int64_t)(g * 16 + 2 * i) * m + ck * MC + 2 * j;
  }

  double acc[IPW][2][NT][2];
#pragma unroll
  for (int u = 0; u < IPW; ++u)
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[u][t][nt][0] = acc[u][t][nt][1] = 0.0;

#pragma unroll
  for (int c = 0; c < NS - 1; ++c) {
    if (c < nch) stage(c);
    else cp_async_commit_group();  // keep the group count uniform
  }
  for (int c = 0; c < nch; ++c) {
    cp_async_wait_groups<NS - 2>();  // chunk c has landed (this thread's copies)
    __syncthreads();                 // ... and everyone's; buffer (c-1) % NS is free
    if (c + NS - 1 < nch) stage(c + NS - 1);
    else cp_async_commit_group();
    const double* buf = stg + (c % NS) * sd;
#pragma unroll
    for (int u = 0; u < IPW; ++u) {
      if (warp + NW * u >= nitems) break;  // warp-uniform
      const double* va = buf + ia[u];
      const double* xb = buf + ib[u];
#pragma unroll
      for (int q = 0; q < R / 4; ++q) {
        const double2 a = *reinterpret_cast<const double2*>(va + q * 4 * VS);
        double bf[NT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) bf[nt] = xb[q * 4 * XS + nt * 8];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          dmma(acc[u][0][nt][0], acc[u][0][nt][1], a.x, bf[nt]);
          dmma(acc[u][1][nt][0], acc[u][1][nt][1], a.y, bf[nt]);
        }
      }
      // node complete (inside the tile) or tile complete (node spans tiles)
      const bool flush = icpn[u] ? ((c + 1) & (icpn[u] - 1)) == 0 : (c == nch - 1);
      if (flush) {
        double* o = iout[u];
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            double* oe = o + (int64_t)e * m + nt * 8;
            if (nt * 8 < icmax[u]) oe[0] = acc[u][e][nt][0];
            if (nt * 8 + 1 < icmax[u]) oe[1] = acc[u][e][nt][1];
            acc[u][e][nt][0] = acc[u][e][nt][1] = 0.0;
          }
        iout[u] += (int64_t)KT * m;  // next node of the level (inside the tile)
      }
    }
  }
  cp_async_wait_groups<0>();
}

// HODLR, nrhs >= 2: tile = LPC leaves (LPC b rows), warp w = leaf w of the tile.
// Per level: warp partial t over its b rows (DMMA), staged in shared memory,
// then fixed-order sums over the warps of each node.
template <int KT, int NT, int LPC = 8>
__global__ void __launch_bounds__(32 * LPC) vt_mma_levels_kernel(const VtParams P, int64_t b) {
  extern __shared__ double red[];  // [LPC][KT][MC]
  constexpr int MC = NT * 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t tile = LPC * b;  // LPC leaves per CTA, one warp each
  const int64_t row0 = (int64_t)blockIdx.x * tile + (int64_t)warp * b;
  const int m = P.m;
  for (int c0 = 0; c0 < m; c0 += MC) {
    const int mc = min(MC, m - c0);
    for (int L = 0; L < P.nlev; ++L) {
      const VtLevel lv = P.lev[L];
      double acc[(KT + 7) / 8][NT][2];
#pragma unroll
      for (int t = 0; t < (KT + 7) / 8; ++t)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[t][nt][0] = acc[t][nt][1] = 0.0;
      if constexpr (KT < 16) {
        warp_transposed_mma_small<KT, NT, (NT > 4 ? 4 : 8)>(acc, lv.V + row0 * KT, P.X + row0 * m, m, c0, m, (int)b,
                                                           lane);
        const int i = lane >> 2, j = lane & 3;
        if (i < KT)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            double* o = red + ((int64_t)warp * KT + i) * MC + nt * 8 + 2 * j;
            o[0] = acc[0][nt][0];
            o[1] = acc[0][nt][1];
          }
      } else {
        warp_transposed_mma<KT / 16, NT, false, HM_VTM_PF(NT)>(acc, lv.V + row0 * KT, KT, P.X + row0 * m, m, c0, m,
                                                               (int)b, lane);
        store_transposed<KT / 16, NT>(acc, red + (int64_t)warp * KT * MC, MC, c0, c0 + mc, lane, c0);
      }
      __syncthreads();
      const int64_t g = lv.s >= tile ? LPC : lv.s / b;
      const int ngroups = (int)(LPC / g);
      for (int o = threadIdx.x; o < ngroups * KT * mc; o += 32 * LPC) {
        const int grp = o / (KT * mc);
        const int rem = o - grp * KT * mc;
        const int a = rem / mc, c = rem - a * mc;
        double s = 0.0;
        for (int w = 0; w < g; ++w) s += red[((int64_t)(grp * g + w) * KT + a) * MC + c];
        const int64_t rfirst = (int64_t)blockIdx.x * tile + grp * g * b;
        if (lv.s > tile) {
          lv.partial[((int64_t)blockIdx.x * KT + a) * m + c0 + c] = s;
        } else {
          lv.out[((rfirst / lv.s) * KT + a) * m + c0 + c] = s;
        }
      }
      __syncthreads();
    }
  }
}

}  // namespace hm
