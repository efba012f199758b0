// hm_leafup.cuh — HSS Step 1 fused with the first upsweep level,
// nrhs >= 2, DMMA:
//
//   x_{p,i}   = V_i^T X(I_i)
//   x_{p-1,q} = W_{p-1,q}^T [x_{p,2q}; x_{p,2q+1}]
//
// Persistent CTAs walk leaf pairs (a level-(p-1) node each). The rows of V_i
// and X(I_i) are staged with cp.async in units of `ru` rows through a 4-slot
// ring (cp.async groups): three units are in flight while one is contracted,
// and the parent's W rides along with the pair's first unit. The pair's two x blocks
// stay in shared memory and feed the parent's W^T product directly; every x
// block is also written to the workspace (the coupling step reads them).
// Fragments: transposed pattern (rows r + (lane&3)) from padded shared rows,
// stride = 4 (mod 16) doubles for the 128-bit A loads and 4 (mod 8) for the
// 64-bit B loads: conflict-free. Each warp owns 16 x 8 output tiles and keeps
// 4 independent accumulator sets over the contraction (k-step mod 4) so
// consecutive DMMAs do not wait on each other; the sets are added in a fixed
// order at the end.
#pragma once
#include "hm_fast.cuh"

namespace hm {

struct LeafUpParams {
  const double* V;  // [n][k] leaf bases
  const double* X;  // [n][m]
  const double* W;  // [2^p-2][2k][k] (level p-1 nodes at 2^(p-1)-2 ..), NULL if p < 2
  double* xh;       // level-major x blocks [.][k][m]
  int64_t npairs;   // 2^(p-1)
  int32_t b, m, p;
  int32_t ru;       // rows per pipeline unit (divides b, multiple of 32)
  int32_t wd;       // depth of the W ring: 2 if a leaf has >= 2 units, else 3
  int32_t pad;
};

// cp.async staging of `rows` rows of COLS doubles (COLS a power of two >= 2,
// compile time, so the chunk -> (row, col) split is a shift and a mask):
// global rows with stride lds, shared rows with stride zs.
template <int COLS>
__device__ __forceinline__ void stage_rows_pow2(double* dst, int zs, const double* src, int64_t lds, int rows) {
  constexpr int H = COLS / 2;  // 16-byte chunks per row
  constexpr int LH = H >= 32 ? 5 : (H >= 16 ? 4 : (H >= 8 ? 3 : (H >= 4 ? 2 : (H >= 2 ? 1 : 0))));
  for (int e = threadIdx.x; e < rows * H; e += blockDim.x) {
    const int r = e >> LH, c = (e & (H - 1)) * 2;
    cp_async16(dst + r * zs + c, src + (int64_t)r * lds + c);
  }
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

constexpr int kLeafUpStages = 4;  // pipeline units in shared memory (3 in flight while one is used)

template <int KT, int MP>
struct LeafUpLayout {
  static constexpr int ZV = KT + 4;  // = 4 (mod 16) for KT in {16, 32, 64}
  static constexpr int ZX = MP + 4;  // = 4 (mod 8)
  static constexpr int MG = KT / 16, CT = MP / 8, TILES = MG * CT;
  __host__ __device__ static constexpr size_t unit_doubles(int ru) { return (size_t)ru * (ZV + ZX); }
  __host__ __device__ static constexpr size_t smem_bytes(int ru, int wd) {
    return sizeof(double) * (kLeafUpStages * unit_doubles(ru) + 2 * (size_t)KT * ZX + (size_t)wd * 2 * KT * ZV +
                             (size_t)TILES * 32 * 8);
  }
};

// C (16 x 8 tile: rank rows 16 g + 2i + e, cols 8 ct + 2j + {0,1}) += A^T B with
// A = As [K][za] (the tile's 16 rank columns at As + 16 g), B = Bs [K][zb]
// (8 columns at Bs + 8 ct); A from shared (ASM) or global memory.
template <bool ASM>
__device__ __forceinline__ void tile_tn(double (&acc)[4][2][2], const double* As, int za, const double* Bs, int zb,
                                        int K, int lane) {
  const int j = lane & 3, i = lane >> 2;
  const double* ap = As + j * za + 2 * i;
  const double* bp = Bs + j * zb + i;
#pragma unroll 1
  for (int q0 = 0; q0 < K / 4; q0 += 4) {  // K % 16 == 0
    double2 a[4];
    double bf[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int q = q0 + s;
      a[s] = ASM ? *reinterpret_cast<const double2*>(ap + q * 4 * za) : ldg_stream2(ap + (int64_t)q * 4 * za);
      bf[s] = bp[q * 4 * zb];
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      dmma(acc[s][0][0], acc[s][0][1], a[s].x, bf[s]);
      dmma(acc[s][1][0], acc[s][1][1], a[s].y, bf[s]);
    }
  }
}

// Sum the 4 accumulator sets (fixed order) and store the tile to shared
// memory (row stride zs) and, if gout != nullptr, to global [.][m].
__device__ __forceinline__ void tile_store(const double (&acc)[4][2][2], int g, int ct, double* sm, int zs,
                                           double* gout, int m, int lane) {
  const int j = lane & 3, i = lane >> 2;
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int a = 16 * g + 2 * i + e;
    const int c = 8 * ct + 2 * j;
    const double v0 = (acc[0][e][0] + acc[1][e][0]) + (acc[2][e][0] + acc[3][e][0]);
    const double v1 = (acc[0][e][1] + acc[1][e][1]) + (acc[2][e][1] + acc[3][e][1]);
    if (sm) {
      sm[a * zs + c] = v0;
      sm[a * zs + c + 1] = v1;
    }
    if (gout) {
      if (c < m) gout[(int64_t)a * m + c] = v0;
      if (c + 1 < m) gout[(int64_t)a * m + c + 1] = v1;
    }
  }
}

// 16 warps: warp w owns tile (w & 7) [+ 8, 16, .. if TILES > 8] over one half of
// every contraction (kh = w >> 3: the first or second half of the unit's rows;
// for the parent, the left or the right child). At the end of a leaf (or of
// the parent) the second half's partial sums go through shared memory and are
// added to the first half's in a fixed order. Accumulators persist over the
// units of a leaf.
constexpr int kLeafUpThreads = 512;

template <int KT, int MP>
__global__ void __launch_bounds__(kLeafUpThreads, 1) hss_leaf_up_kernel(const LeafUpParams P) {
  using L = LeafUpLayout<KT, MP>;
  constexpr int TPW = (L::TILES + 7) / 8;  // tiles per warp
  constexpr int NS = kLeafUpStages;
  extern __shared__ __align__(16) double lsm[];
  const int b = P.b, m = P.m, ru = P.ru;
  const int upl = b / ru;  // units per leaf
  double* xs = lsm + NS * L::unit_doubles(ru);  // [2][KT][ZX]: the pair's x blocks
  // [wd][2KT][ZV]: W of the pair's parent. Pair P's W is staged NS-1 = 3 units
  // before the pair starts and read after its last unit (2 upl units later):
  // pair P+wd's staging comes after that use iff 2 upl wd > 2 upl + 2, i.e.
  // wd = 2 for upl >= 2 and wd = 3 for upl = 1.
  const int wd = P.wd;
  double* wring = xs + 2 * KT * L::ZX;
  double* red = wring + (size_t)wd * 2 * KT * L::ZV;  // [TILES][32 lanes][8]: second-half partials
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wt = warp & 7, kh = warp >> 3;
  const int64_t km = (int64_t)KT * m;
  double* xleaf = P.xh + (((int64_t)1 << P.p) - 2) * km;
  double* xpar = P.p >= 2 ? P.xh + (((int64_t)1 << (P.p - 1)) - 2) * km : nullptr;
  const int64_t npairs = P.npairs;
  const int mypairs = blockIdx.x < npairs ? (int)((npairs - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  const int nunits = 2 * mypairs * upl;
  auto leaf_of = [&](int t) { return 2 * ((int64_t)blockIdx.x + (int64_t)(t >> 1) * gridDim.x) + (t & 1); };
  // staging cursor: unit su = (leaf st of this CTA's list, unit sui of the leaf), advanced incrementally
  int su = 0, st = 0, sui = 0;
  auto stage = [&]() {
    const int r0 = sui * ru;
    const int64_t leaf = leaf_of(st);
    double* s = lsm + (su & (NS - 1)) * L::unit_doubles(ru);
    stage_rows_pow2<KT>(s, L::ZV, P.V + (leaf * b + r0) * KT, KT, ru);
    if (m == MP) stage_rows_pow2<MP>(s + (size_t)ru * L::ZV, L::ZX, P.X + (leaf * b + r0) * m, m, ru);
    else stage_rows_async(s + (size_t)ru * L::ZV, L::ZX, P.X + (leaf * b + r0) * m, m, ru, m, MP);
    if (xpar && (st & 1) == 0 && sui == 0)  // first unit of a pair: the parent's W rides along
      stage_rows_pow2<KT>(wring + ((st >> 1) % wd) * 2 * KT * L::ZV, L::ZV,
                          P.W + (((int64_t)1 << (P.p - 1)) - 2 + (leaf >> 1)) * 2 * KT * KT, KT, 2 * KT);
    ++su;
    if (++sui == upl) { sui = 0; ++st; }
  };
  // second-half partials -> shared; first half adds them (fixed order) and stores
  auto combine_store = [&](double (&acc)[4][2][2], int tile, double* sm, int zs, double* gout) {
    double* rb = red + ((size_t)tile * 32 + lane) * 8;
    if (kh == 1) {
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          rb[e * 2 + h] = (acc[0][e][h] + acc[1][e][h]) + (acc[2][e][h] + acc[3][e][h]);
    }
    __syncthreads();
    if (kh == 0) {
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          acc[0][e][h] = (acc[0][e][h] + acc[1][e][h]) + (acc[2][e][h] + acc[3][e][h]);
          acc[1][e][h] = rb[e * 2 + h];
          acc[2][e][h] = 0.0;
          acc[3][e][h] = 0.0;
        }
      tile_store(acc, tile % L::MG, tile / L::MG, sm, zs, gout, m, lane);
    }
  };
  static_assert((NS & (NS - 1)) == 0, "ring size must be a power of two");
  for (int u = 0; u < NS - 1; ++u) {
    if (u < nunits) stage();
    cp_async_commit();
  }
  double acc[TPW][4][2][2];
  const int hr = ru / 2;  // rows per contraction half
  int t = 0, ui = 0;      // leaf of the list, unit of the leaf (of unit u)
  for (int u = 0; u < nunits; ++u, ++ui == upl ? (ui = 0, ++t) : 0) {
    if (u + NS - 1 < nunits) stage();
    cp_async_commit();
    asm volatile("cp.async.wait_group %0;" ::"n"(NS - 1) : "memory");
    __syncthreads();  // unit u (and, with the pair's first unit, W) staged
    if (ui == 0) {
#pragma unroll
      for (int x = 0; x < TPW; ++x)
#pragma unroll
        for (int s4 = 0; s4 < 4; ++s4)
          acc[x][s4][0][0] = acc[x][s4][0][1] = acc[x][s4][1][0] = acc[x][s4][1][1] = 0.0;
    }
    const double* Vs = lsm + (u & (NS - 1)) * L::unit_doubles(ru) + (size_t)kh * hr * L::ZV;
    const double* Xs = lsm + (u & (NS - 1)) * L::unit_doubles(ru) + (size_t)ru * L::ZV + (size_t)kh * hr * L::ZX;
#pragma unroll
    for (int x = 0; x < TPW; ++x) {
      const int tile = wt + 8 * x;
      if (tile < L::TILES)
        tile_tn<true>(acc[x], Vs + 16 * (tile % L::MG), L::ZV, Xs + 8 * (tile / L::MG), L::ZX, hr, lane);
    }
    if (ui == upl - 1) {  // leaf complete: x to shared (pair slot t & 1) and to the workspace
      const int64_t leaf = leaf_of(t);
#pragma unroll
      for (int x = 0; x < TPW; ++x) {
        const int tile = wt + 8 * x;
        if (tile < L::TILES) combine_store(acc[x], tile, xs + (t & 1) * KT * L::ZX, L::ZX, xleaf + leaf * km);
        else __syncthreads();
      }
    }
    __syncthreads();  // unit slot reusable; xs complete
    if (ui == upl - 1 && (t & 1) && xpar) {  // parent: W^T [x_left; x_right], halves = the two children
      const int64_t q = leaf_of(t) >> 1;
      const double* Wb = wring + ((t >> 1) % wd) * 2 * KT * L::ZV + (size_t)kh * KT * L::ZV;
      const double* Xb = xs + (size_t)kh * KT * L::ZX;
#pragma unroll
      for (int x = 0; x < TPW; ++x) {
        const int tile = wt + 8 * x;
        double pacc[4][2][2] = {};
        if (tile < L::TILES) {
          tile_tn<true>(pacc, Wb + 16 * (tile % L::MG), L::ZV, Xb + 8 * (tile / L::MG), L::ZX, KT, lane);
          combine_store(pacc, tile, nullptr, 0, xpar + q * km);
        } else {
          __syncthreads();
        }
      }
      __syncthreads();  // xs reusable
    }
  }
  cp_async_wait_all();
}

}  // namespace hm
