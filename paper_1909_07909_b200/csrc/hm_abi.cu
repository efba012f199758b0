// hm_abi.cu — the C-ABI of libhm (include/hm.h): host-side validation,
// workspace layout and kernel launches for the HODLR / HSS matvec.
//
// Paper: hm-toolbox (arXiv 1909.07909); "P:n" = line n of PAPER.md.
// Validation happens entirely on the host before the first launch, so a
// negative status means nothing was enqueued (except HM_ERR_CUDA).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hm.h"
#include "hm_kernels.cuh"
#include "hm_fast.cuh"
#include "hm_tree.cuh"

namespace {

thread_local std::string g_err;
thread_local int32_t g_launches = 0;

hm_status fail(hm_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

hm_status cuda_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HM_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return HM_OK;
}

// ----------------------------------------------------------- launch trace --
// hm_profile_enable / hm_profile_collect: every launch bracketed by two events.
struct TraceRec {
  const char* name;
  int32_t call;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
int32_t g_prof_call = -1;
std::vector<TraceRec> g_prof_recs;
std::vector<cudaEvent_t> g_prof_pool;

cudaEvent_t prof_event() {
  if (!g_prof_pool.empty()) {
    cudaEvent_t e = g_prof_pool.back();
    g_prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

void prof_new_call() {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (g_prof_on) ++g_prof_call;
}

// Records the start event; returns the trace slot (or -1 when tracing is off).
int prof_begin(const char* name, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (!g_prof_on) return -1;
  TraceRec r{name, g_prof_call, prof_event(), prof_event()};
  cudaEventRecord(r.a, s);
  g_prof_recs.push_back(r);
  return (int)g_prof_recs.size() - 1;
}

void prof_end(int slot, cudaStream_t s) {
  if (slot < 0) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (slot < (int)g_prof_recs.size()) cudaEventRecord(g_prof_recs[slot].b, s);
}

constexpr size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Columns of X handled per CTA, and the leaf-group tile of vt_contract.
constexpr int64_t kSmemBudgetDoubles = 160 * 1024 / 8;  // 160 KB of dynamic smem
constexpr int64_t kTileDoubles = 4096;                    // X tile of vt_contract: 32 KB

int pick_mc(int64_t b, int64_t ktot, int32_t m) {
  int mc = 1;
  while (mc < hm::kMaxMc && mc < m) mc <<= 1;
  while (mc > 1 && (b + ktot) * mc > kSmemBudgetDoubles) mc >>= 1;
  return mc;
}

int vt_mc(int64_t b, int32_t m) {
  int mc = std::min<int32_t>(m, hm::kMaxMc);
  while (mc > 1 && b * mc + hm::kThreads > kSmemBudgetDoubles) --mc;
  return mc;
}

// tile = b * 2^i (i <= p) with tile * mc <= kTileDoubles when possible: every
// node size s_l = b 2^{p-l} then divides or is divided by the tile.
int64_t pick_tile(int64_t b, int32_t p, int32_t mc) {
  int64_t tile = b;
  int i = 0;
  while (i < p && tile * 2 * mc <= kTileDoubles) { tile *= 2; ++i; }
  return tile;
}

hm_status check_tree(const hm_tree* t) {
  if (!t) return fail(HM_ERR_INVALID_ARG, "tree is NULL");
  if (t->flags != 0) return fail(HM_ERR_UNSUPPORTED, "tree flags %d: only the balanced tree of P:86-91 is built", t->flags);
  if (t->n < 1 || t->leaf < 1 || t->levels < 0 || t->levels > 40)
    return fail(HM_ERR_INVALID_ARG, "tree: need n >= 1, leaf >= 1, 0 <= levels <= 40 (n=%lld leaf=%lld levels=%d)",
                (long long)t->n, (long long)t->leaf, t->levels);
  if ((t->leaf << t->levels) != t->n)
    return fail(HM_ERR_UNSUPPORTED, "n = %lld is not leaf * 2^levels = %lld * 2^%d (general endpoint vectors, P:560-565, not built)",
                (long long)t->n, (long long)t->leaf, t->levels);
  if (t->leaf + hm::kMaxRank * t->levels > kSmemBudgetDoubles)
    return fail(HM_ERR_UNSUPPORTED, "leaf size %lld exceeds the shared-memory staging limit", (long long)t->leaf);
  if (t->levels + 1 > hm::kMaxLevels) return fail(HM_ERR_UNSUPPORTED, "too many levels");
  return HM_OK;
}

bool overlap(const void* a, size_t na, const void* b, size_t nb) {
  auto x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
  return x < y + nb && y < x + na;
}

// ---------------------------------------------------------------- dispatch --
#ifndef HM_VTB_NTMAX
#define HM_VTB_NTMAX 4
#endif
#ifndef HM_TREE_NTMAX
#define HM_TREE_NTMAX 4
#endif
// Which kernels run is decided on the host from the shapes:
// the tuned kernels of hm_fast.cuh where their shape conditions hold, the
// generic kernels of hm_kernels.cuh otherwise. Both are exact implementations
// of the same steps; the parity tests cover both families.

bool pow2_rank(int k, int lo, int hi) {
  for (int v = lo; v <= hi; v <<= 1)
    if (k == v) return true;
  return false;
}

int nt_for(int m, int cap) {
  int nt = 1;
  while (nt < cap && nt * 8 < m) nt <<= 1;
  return nt;
}

template <typename F>
hm_status launch(const char* name, cudaStream_t s, F&& f) {
  int slot = prof_begin(name, s);
  f();
  prof_end(slot, s);
  ++g_launches;
  return cuda_check(name);
}

template <typename K>
void allow_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// ------------------------------------------------------------------ HODLR --

enum class VtPath { kNone, kGeneric, kGemv, kMma };
enum class LeafPath { kGeneric, kGemv, kMma };

struct HodlrPlan {
  int64_t n, b;
  int32_t p, m, k;  // k = the common nonzero rank (0 if all zero)
  int64_t ktot;
  VtPath vt;
  LeafPath leaf;
  int32_t mc_vt, mc_leaf, nt_vt, nt_leaf;
  int64_t tile;  // rows per vt CTA
  size_t off_t[hm::kMaxLevels + 1];
  size_t off_part[hm::kMaxLevels + 1];
  size_t off_x, off_y, total;
};

hm_status hodlr_plan(const hm_tree* tree, const int32_t* ranks, int32_t nrhs, int32_t flags, HodlrPlan* P) {
  hm_status st = check_tree(tree);
  if (st) return st;
  if (nrhs < 1) return fail(HM_ERR_INVALID_ARG, "nrhs = %d < 1", nrhs);
  if (tree->levels > 0 && !ranks) return fail(HM_ERR_INVALID_ARG, "ranks is NULL");
  memset(P, 0, sizeof *P);
  P->n = tree->n; P->b = tree->leaf; P->p = tree->levels; P->m = nrhs;
  for (int l = 1; l <= P->p; ++l) {
    int k = ranks[l - 1];
    if (k < 0) return fail(HM_ERR_INVALID_ARG, "ranks[%d] = %d < 0", l - 1, k);
    if (k > hm::kMaxRank) return fail(HM_ERR_UNSUPPORTED, "rank %d > %d", k, hm::kMaxRank);
    if (k > 0) {
      if (P->k != 0 && P->k != k)
        return fail(HM_ERR_UNSUPPORTED, "per-level ranks differ (%d vs %d); variable ranks (P:264) not built", P->k, k);
      P->k = k;
    }
    P->ktot += k;
  }
  const int64_t b = P->b, k = P->k;
  const bool tiles8 = P->p >= 3;  // 8-leaf row tiles exist
  // phase 1: V_l^T X
  if (k == 0 || P->p == 0) {
    P->vt = VtPath::kNone;
  } else if (nrhs == 1 && tiles8 && b % 64 == 0 && b <= 4096 && pow2_rank((int)k, 1, 64)) {
    P->vt = VtPath::kGemv;
    P->tile = 8 * b;
  } else if (nrhs >= 2 && tiles8 && b % 4 == 0 && pow2_rank((int)k, 16, 64)) {
    P->vt = VtPath::kMma;
    P->tile = 8 * b;
    P->nt_vt = nt_for(nrhs, k == 64 ? 2 : 4);
  } else {
    P->vt = VtPath::kGeneric;
    P->mc_vt = vt_mc(b, nrhs);
    P->tile = pick_tile(b, P->p, P->mc_vt);
  }
  // phase 2: leaves
  const bool k8 = (k % 8 == 0);
  if (nrhs == 1 && b % 64 == 0 && b <= 1024 && (k == 0 || pow2_rank((int)k, 1, 64)) &&
      (2 * b + P->ktot) * 8 <= 160 * 1024) {
    P->leaf = LeafPath::kGemv;
  } else if (nrhs >= 2 && (b == 64 || b == 128 || b == 256) && k8) {
    P->leaf = LeafPath::kMma;
    const int rg = (int)(b / 64);
    P->nt_leaf = nt_for(nrhs, rg == 4 ? 2 : 4);
    if ((b + P->ktot) * (8 * P->nt_leaf + 4) > kSmemBudgetDoubles) P->leaf = LeafPath::kGeneric;
  } else {
    P->leaf = LeafPath::kGeneric;
  }
  if (P->leaf == LeafPath::kGeneric) {
    P->mc_leaf = pick_mc(b, P->ktot, nrhs);
    if ((b + P->ktot) * P->mc_leaf > kSmemBudgetDoubles)
      return fail(HM_ERR_UNSUPPORTED, "leaf %lld + ranks %lld too large for shared-memory staging", (long long)b,
                  (long long)P->ktot);
  }
  // workspace: t_l per level, per-tile partials where a node spans several tiles
  size_t off = 0;
  for (int l = 1; l <= P->p; ++l) {
    P->off_t[l] = off;
    off = align_up(off + sizeof(double) * (size_t)((1ll << l) * ranks[l - 1] * nrhs));
  }
  for (int l = 1; l <= P->p; ++l) {
    const int64_t s = P->n >> l;
    P->off_part[l] = off;
    if (P->vt != VtPath::kNone && ranks[l - 1] > 0 && s > P->tile)
      off = align_up(off + sizeof(double) * (size_t)((P->n / P->tile) * ranks[l - 1] * nrhs));
  }
  P->off_x = P->off_y = off;
  if (flags & HM_WS_HOSTIO) {
    P->off_x = off;
    off = align_up(off + sizeof(double) * (size_t)(P->n * nrhs));
    P->off_y = off;
    off = align_up(off + sizeof(double) * (size_t)(P->n * nrhs));
  }
  P->total = std::max<size_t>(off, kAlign);
  return HM_OK;
}

// ---- leaf launches (shared by HODLR and HSS) ----

template <int MC>
hm_status launch_leaf_generic(const hm::LeafParams& lp, int64_t nleaves, cudaStream_t s) {
  size_t smem = sizeof(double) * (size_t)((lp.b + lp.ktot) * MC);
  allow_smem(hm::leaf_apply_kernel<MC>, smem);
  dim3 grid((unsigned)nleaves, (unsigned)((lp.m + MC - 1) / MC));
  return launch("leaf_apply", s, [&] { hm::leaf_apply_kernel<MC><<<grid, hm::kThreads, smem, s>>>(lp); });
}

template <int K>
hm_status launch_leaf_gemv(const hm::LeafParams& lp, int64_t nleaves, cudaStream_t s) {
  size_t smem = sizeof(double) * (size_t)(2 * lp.b + lp.nseg * K);
  allow_smem(hm::leaf_gemv_kernel<K>, smem);
  return launch("leaf_apply", s, [&] { hm::leaf_gemv_kernel<K><<<(unsigned)nleaves, 256, smem, s>>>(lp); });
}

// (RG, NT) -> prefetch depth and launch-bound occupancy (measured, r01_tuning.md)
template <int RG, int NT>
struct LeafMmaTune {
  static constexpr int PF = (RG == 2 && NT == 4) ? 1 : 2;
  static constexpr int MINB = (RG == 2 && NT == 4) ? 4 : 0;
};

template <int RG, int NT>
hm_status launch_leaf_mma(const hm::LeafParams& lp, int64_t nleaves, cudaStream_t s) {
  constexpr int PF = LeafMmaTune<RG, NT>::PF, MINB = LeafMmaTune<RG, NT>::MINB;
  size_t smem = sizeof(double) * (size_t)((lp.b + lp.ktot) * (NT * 8 + 4));
  allow_smem(hm::leaf_mma_kernel<RG, NT, PF, MINB>, smem);
  const int64_t chunks = (lp.m + NT * 8 - 1) / (NT * 8);
  return launch("leaf_apply", s, [&] {
    hm::leaf_mma_kernel<RG, NT, PF, MINB><<<(unsigned)(nleaves * chunks), 256, smem, s>>>(lp);
  });
}

hm_status leaf_dispatch(const hm::LeafParams& lp, int64_t nleaves, LeafPath path, int k, int nt, int mc,
                        cudaStream_t s) {
  if (path == LeafPath::kGemv) {
    switch (k) {
      case 0: case 1: return launch_leaf_gemv<1>(lp, nleaves, s);
      case 2: return launch_leaf_gemv<2>(lp, nleaves, s);
      case 4: return launch_leaf_gemv<4>(lp, nleaves, s);
      case 8: return launch_leaf_gemv<8>(lp, nleaves, s);
      case 16: return launch_leaf_gemv<16>(lp, nleaves, s);
      case 32: return launch_leaf_gemv<32>(lp, nleaves, s);
      default: return launch_leaf_gemv<64>(lp, nleaves, s);
    }
  }
  if (path == LeafPath::kMma) {
    const int rg = (int)(lp.b / 64);
#define HM_LEAF_MMA(RG_)                                            \
  if (rg == RG_) {                                                  \
    if (nt == 1) return launch_leaf_mma<RG_, 1>(lp, nleaves, s);    \
    if (nt == 2) return launch_leaf_mma<RG_, 2>(lp, nleaves, s);    \
    if constexpr (RG_ < 4) return launch_leaf_mma<RG_, 4>(lp, nleaves, s); \
  }
    HM_LEAF_MMA(1)
    HM_LEAF_MMA(2)
    HM_LEAF_MMA(4)
#undef HM_LEAF_MMA
    return fail(HM_ERR_UNSUPPORTED, "leaf_mma: no instance for b=%lld nt=%d", (long long)lp.b, nt);
  }
  switch (mc) {
    case 1: return launch_leaf_generic<1>(lp, nleaves, s);
    case 2: return launch_leaf_generic<2>(lp, nleaves, s);
    case 4: return launch_leaf_generic<4>(lp, nleaves, s);
    case 8: return launch_leaf_generic<8>(lp, nleaves, s);
    default: return launch_leaf_generic<16>(lp, nleaves, s);
  }
}

// ---- V^T X launches ----

hm_status vt_generic(const hm::VtParams& vp, int64_t n, cudaStream_t s) {
  size_t smem = sizeof(double) * (size_t)(vp.tile * vp.mc + hm::kThreads);
  allow_smem(hm::vt_contract_kernel, smem);
  dim3 grid((unsigned)(n / vp.tile), (unsigned)((vp.m + vp.mc - 1) / vp.mc));
  return launch("vt_contract", s, [&] { hm::vt_contract_kernel<<<grid, hm::kThreads, smem, s>>>(vp); });
}

template <int K>
hm_status vt_gemv_launch(const hm::VtParams& vp, int64_t b, cudaStream_t s) {
  hm::VtGemvParams gp;
  memset(&gp, 0, sizeof gp);
  gp.X = vp.X; gp.n = vp.n; gp.b = b; gp.nlev = vp.nlev;
  for (int i = 0; i < vp.nlev; ++i) gp.lev[i] = vp.lev[i];
  size_t smem = sizeof(double) * (size_t)(8 * b);
  allow_smem(hm::vt_gemv_kernel<K>, smem);
  return launch("vt_contract", s,
                [&] { hm::vt_gemv_kernel<K><<<(unsigned)(vp.n / (8 * b)), 256, smem, s>>>(gp); });
}

hm_status vt_gemv_dispatch(const hm::VtParams& vp, int64_t b, int k, cudaStream_t s) {
  switch (k) {
    case 1: return vt_gemv_launch<1>(vp, b, s);
    case 2: return vt_gemv_launch<2>(vp, b, s);
    case 4: return vt_gemv_launch<4>(vp, b, s);
    case 8: return vt_gemv_launch<8>(vp, b, s);
    case 16: return vt_gemv_launch<16>(vp, b, s);
    case 32: return vt_gemv_launch<32>(vp, b, s);
    default: return vt_gemv_launch<64>(vp, b, s);
  }
}

template <int KT, int NT>
hm_status vt_mma_launch(const hm::VtParams& vp, int64_t b, cudaStream_t s) {
  size_t smem = sizeof(double) * (size_t)(8 * KT * NT * 8);
  allow_smem(hm::vt_mma_levels_kernel<KT, NT>, smem);
  return launch("vt_contract", s, [&] {
    hm::vt_mma_levels_kernel<KT, NT><<<(unsigned)(vp.n / (8 * b)), 256, smem, s>>>(vp, b);
  });
}

hm_status vt_mma_dispatch(const hm::VtParams& vp, int64_t b, int k, int nt, cudaStream_t s) {
#define HM_VT_MMA(KT_)                                             \
  if (k == KT_) {                                                  \
    if (nt == 1) return vt_mma_launch<KT_, 1>(vp, b, s);           \
    if (nt == 2) return vt_mma_launch<KT_, 2>(vp, b, s);           \
    if constexpr (KT_ < 64) return vt_mma_launch<KT_, 4>(vp, b, s); \
  }
  HM_VT_MMA(16)
  HM_VT_MMA(32)
  HM_VT_MMA(64)
#undef HM_VT_MMA
  return fail(HM_ERR_UNSUPPORTED, "vt_mma: no instance for k=%d nt=%d", k, nt);
}

template <int KT, int NT>
hm_status vt_batched_launch(const char* name, const hm::BatchedVtParams& bp, cudaStream_t s) {
  constexpr int MPW = 1;
  const int64_t nck = (bp.m + NT * 8 - 1) / (NT * 8);
  const int64_t warps = bp.count * (KT / 16 / MPW) * nck;
  return launch(name, s, [&] {
    hm::vt_batched_kernel<KT, MPW, NT><<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(bp);
  });
}

hm_status vt_batched_dispatch(const char* name, const hm::BatchedVtParams& bp, int k, int nt, cudaStream_t s) {
#define HM_VTB(KT_)                                                 \
  if (k == KT_) {                                                   \
    if (nt == 1) return vt_batched_launch<KT_, 1>(name, bp, s);     \
    if (nt == 2) return vt_batched_launch<KT_, 2>(name, bp, s);     \
    return vt_batched_launch<KT_, 4>(name, bp, s);                  \
  }
  HM_VTB(16)
  HM_VTB(32)
  HM_VTB(64)
#undef HM_VTB
  return fail(HM_ERR_UNSUPPORTED, "vt_batched: no instance for k=%d nt=%d", k, nt);
}

hm_status hodlr_run(const hm_tree* tree, const int32_t* ranks, const double* D, const double* U,
                    const double* V, const double* X, int32_t nrhs, double* Y, void* ws, size_t ws_bytes,
                    cudaStream_t stream, int32_t flags) {
  HodlrPlan P;
  hm_status st = hodlr_plan(tree, ranks, nrhs, flags, &P);
  if (st) return st;
  if (!ws || ws_bytes < P.total)
    return fail(HM_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, P.total);
  if (!D || !X || !Y || (P.k > 0 && (!U || !V)))
    return fail(HM_ERR_INVALID_ARG, "NULL generator / X / Y pointer");
  if (!aligned16(D) || !aligned16(ws) || (P.k > 0 && (!aligned16(U) || !aligned16(V))))
    return fail(HM_ERR_INVALID_ARG, "D, U, V and the workspace must be 16-byte aligned");
  const size_t xy_bytes = sizeof(double) * (size_t)(P.n * nrhs);
  if (overlap(X, xy_bytes, Y, xy_bytes)) return fail(HM_ERR_INVALID_ARG, "X and Y overlap");
  if (!(flags & HM_WS_HOSTIO) && (!aligned16(X) || !aligned16(Y)))
    return fail(HM_ERR_INVALID_ARG, "X and Y must be 16-byte aligned");

  char* w = static_cast<char*>(ws);
  const double* Xd = X;
  double* Yd = Y;
  g_launches = 0;
  prof_new_call();
  if (flags & HM_WS_HOSTIO) {
    Xd = reinterpret_cast<double*>(w + P.off_x);
    Yd = reinterpret_cast<double*>(w + P.off_y);
    if (cudaMemcpyAsync(const_cast<double*>(Xd), X, xy_bytes, cudaMemcpyHostToDevice, stream) != cudaSuccess)
      return cuda_check("H2D copy of X");
  }

  // (1) every level's V_l^T X in one pass over row tiles; partials -> fixed-order reduce
  if (P.vt != VtPath::kNone) {
    hm::VtParams vp;
    memset(&vp, 0, sizeof vp);
    vp.X = Xd; vp.n = P.n; vp.m = nrhs; vp.mc = P.mc_vt; vp.tile = P.tile;
    hm::ReduceParams rp;
    memset(&rp, 0, sizeof rp);
    int64_t uoff = 0;
    for (int l = 1; l <= P.p; ++l) {
      const int k = ranks[l - 1];
      const int64_t s = P.n >> l;
      if (k > 0) {
        hm::VtLevel& lv = vp.lev[vp.nlev++];
        lv.V = V + uoff;
        lv.k = k;
        lv.s = s;
        lv.out = reinterpret_cast<double*>(w + P.off_t[l]);
        lv.partial = reinterpret_cast<double*>(w + P.off_part[l]);
        if (s > P.tile) {
          hm::ReduceLevel& rl = rp.lev[rp.nlev++];
          rl.partial = lv.partial;
          rl.out = lv.out;
          rl.nodes = 1ll << l;
          rl.per_node = (int32_t)(s / P.tile);
          rl.km = k * nrhs;
          int lg = 0;
          while (lg < 5 && (1 << lg) < rl.per_node / 4) ++lg;  // ~4+ partials per lane
          rl.log2g = lg;
          rl.thread_begin = rp.threads;
          rp.threads += ((rl.nodes * rl.km << lg) + 31) / 32 * 32;
        }
      }
      uoff += P.n * k;
    }
    if (P.vt == VtPath::kGemv) st = vt_gemv_dispatch(vp, P.b, P.k, stream);
    else if (P.vt == VtPath::kMma) st = vt_mma_dispatch(vp, P.b, P.k, P.nt_vt, stream);
    else st = vt_generic(vp, P.n, stream);
    if (st) return st;
    if (rp.nlev > 0) {
      const unsigned grid = (unsigned)((rp.threads + hm::kThreads - 1) / hm::kThreads);
      st = launch("reduce_partials", stream,
                  [&] { hm::reduce_partials_kernel<<<grid, hm::kThreads, 0, stream>>>(rp); });
      if (st) return st;
    }
  }

  // (2) per leaf: Y(I_i) = D_i X(I_i) + sum_l U_l(I_i) t_{l, sib(node_l(i))}
  hm::LeafParams lp;
  memset(&lp, 0, sizeof lp);
  lp.D = D; lp.X = Xd; lp.Y = Yd; lp.b = P.b; lp.m = nrhs; lp.mc = P.mc_leaf;
  {
    int64_t uoff = 0;
    for (int l = 1; l <= P.p; ++l) {
      const int k = ranks[l - 1];
      if (k > 0) {
        hm::LeafSeg& sg = lp.seg[lp.nseg++];
        sg.A = U + uoff;
        sg.T = reinterpret_cast<const double*>(w + P.off_t[l]);
        sg.k = k;
        sg.shift = P.p - l;  // node of leaf i at level l: i >> (p - l)
        sg.xr = 1;           // the sibling's coefficients: A(I_a, I_sib a) = U(I_a) V(I_sib)^T
        lp.ktot += k;
      }
      uoff += P.n * k;
    }
  }
  if ((st = leaf_dispatch(lp, 1ll << P.p, P.leaf, P.k, P.nt_leaf, P.mc_leaf, stream))) return st;

  if (flags & HM_WS_HOSTIO) {
    if (cudaMemcpyAsync(Y, Yd, xy_bytes, cudaMemcpyDeviceToHost, stream) != cudaSuccess)
      return cuda_check("D2H copy of Y");
  }
  return HM_OK;
}

// -------------------------------------------------------------------- HSS --

struct HssPlan {
  int64_t n, b;
  int32_t p, m, k;
  VtPath vt;
  LeafPath leaf;
  bool mma_levels;  // DMMA up/down level kernels
  int32_t mc_vt, mc_leaf, nt_vt, nt_leaf, nt_down;
  int64_t tile;
  size_t off_xh, off_yh, off_x, off_y, total;
};

hm_status hss_plan(const hm_tree* tree, int32_t k, int32_t nrhs, int32_t flags, HssPlan* P) {
  hm_status st = check_tree(tree);
  if (st) return st;
  if (nrhs < 1) return fail(HM_ERR_INVALID_ARG, "nrhs = %d < 1", nrhs);
  if (k < 0) return fail(HM_ERR_INVALID_ARG, "k = %d < 0", k);
  if (k > hm::kMaxRank) return fail(HM_ERR_UNSUPPORTED, "rank %d > %d", k, hm::kMaxRank);
  memset(P, 0, sizeof *P);
  P->n = tree->n; P->b = tree->leaf; P->p = tree->levels; P->m = nrhs; P->k = k;
  const int64_t b = P->b;
  const bool coupled = (k > 0 && P->p > 0);
  if (!coupled) {
    P->vt = VtPath::kNone;
  } else if (nrhs == 1 && P->p >= 3 && b % 64 == 0 && b <= 4096 && pow2_rank(k, 1, 64)) {
    P->vt = VtPath::kGemv;
    P->tile = 8 * b;
  } else if (nrhs >= 2 && b % 4 == 0 && pow2_rank(k, 16, 64)) {
    P->vt = VtPath::kMma;  // batched: one warp per leaf
    P->nt_vt = nt_for(nrhs, HM_VTB_NTMAX);
  } else {
    P->vt = VtPath::kGeneric;
    P->mc_vt = vt_mc(b, nrhs);
    P->tile = pick_tile(b, P->p, P->mc_vt);
  }
  P->mma_levels = coupled && nrhs >= 2 && pow2_rank(k, 16, 64);
  if (P->mma_levels) P->nt_down = nt_for(nrhs, HM_TREE_NTMAX);
  const int ktot = coupled ? k : 0;
  if (nrhs == 1 && b % 64 == 0 && b <= 1024 && (ktot == 0 || pow2_rank(ktot, 1, 64))) {
    P->leaf = LeafPath::kGemv;
  } else if (nrhs >= 2 && (b == 64 || b == 128 || b == 256) && ktot % 8 == 0) {
    P->leaf = LeafPath::kMma;
    P->nt_leaf = nt_for(nrhs, b == 256 ? 2 : 4);
    if ((b + ktot) * (8 * P->nt_leaf + 4) > kSmemBudgetDoubles) P->leaf = LeafPath::kGeneric;
  } else {
    P->leaf = LeafPath::kGeneric;
  }
  if (P->leaf == LeafPath::kGeneric) {
    P->mc_leaf = pick_mc(b, ktot, nrhs);
    if ((b + ktot) * P->mc_leaf > kSmemBudgetDoubles)
      return fail(HM_ERR_UNSUPPORTED, "leaf %lld too large for shared-memory staging", (long long)b);
  }
  const size_t coef = sizeof(double) * (size_t)((((int64_t)1 << (P->p + 1)) - 2) * k * nrhs);
  size_t off = 0;
  P->off_xh = off; off = align_up(off + coef);
  P->off_yh = off; off = align_up(off + coef);
  P->off_x = P->off_y = off;
  if (flags & HM_WS_HOSTIO) {
    P->off_x = off; off = align_up(off + sizeof(double) * (size_t)(P->n * nrhs));
    P->off_y = off; off = align_up(off + sizeof(double) * (size_t)(P->n * nrhs));
  }
  P->total = std::max<size_t>(off, kAlign);
  return HM_OK;
}

template <int KT, int NT>
hm_status hss_down_launch(const hm::HssDownParams& dp, cudaStream_t s) {
  const int64_t cnt = 1ll << dp.level;
  const int64_t nck = (dp.m + NT * 8 - 1) / (NT * 8);
  const int64_t warps = cnt * (KT / 8) * nck;
  return launch("hss_down_level", s,
                [&] { hm::hss_down_mma_kernel<KT, NT><<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(dp); });
}

hm_status hss_down_dispatch(const hm::HssDownParams& dp, int k, int nt, cudaStream_t s) {
#define HM_DOWN(KT_)                                              \
  if (k == KT_) {                                                 \
    if (nt == 1) return hss_down_launch<KT_, 1>(dp, s);           \
    if (nt == 2) return hss_down_launch<KT_, 2>(dp, s);           \
    return hss_down_launch<KT_, 4>(dp, s);                        \
  }
  HM_DOWN(16)
  HM_DOWN(32)
  HM_DOWN(64)
#undef HM_DOWN
  return fail(HM_ERR_UNSUPPORTED, "hss_down: no instance for k=%d nt=%d", k, nt);
}

// Levels with at least kTreeBigLevel nodes run one launch per level; the
// levels above run inside one cooperative launch (hss_tree_sweep_kernel).
constexpr int64_t kTreeBigLevel = 2048;

template <int KT, int NT>
hm_status tree_launch(const hm::TreeParams& tp, int p, cudaStream_t s) {
  constexpr int MINB = (KT == 32 && NT == 4) ? 3 : 0;  // measured, r01_tuning.md
  const size_t smem = sizeof(double) * (size_t)hm::tree_smem_doubles(KT, tp.m, NT);
  static bool attrs = false;
  int sweep_blocks_per_sm = 0;
  if (!attrs) {
    allow_smem(hm::hss_up_pair_kernel<KT, NT, MINB>, 200 * 1024);
    allow_smem(hm::hss_down_pair_kernel<KT, NT, MINB>, 200 * 1024);
    allow_smem(hm::hss_tree_sweep_kernel<KT, NT>, 200 * 1024);
    attrs = true;
  }
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&sweep_blocks_per_sm, hm::hss_tree_sweep_kernel<KT, NT>, 256,
                                                    smem) != cudaSuccess)
    return cuda_check("occupancy query (hss_tree_sweep)");
  int lbig = 1;  // first level with >= kTreeBigLevel nodes
  while (lbig <= p && (1ll << lbig) < kTreeBigLevel) ++lbig;
  hm_status st;
  // upsweep: big levels p-1 .. lbig one launch each
  for (int l = p - 1; l >= lbig; --l) {
    const unsigned pairs = (unsigned)(1ll << (l - 1));
    st = launch("hss_up_level", s, [&] { hm::hss_up_pair_kernel<KT, NT, MINB><<<pairs, 256, smem, s>>>(tp, l); });
    if (st) return st;
  }
  // small levels: up min(p-1, lbig-1) .. 1, down 1 .. min(p, lbig-1)
  const int up_from = std::min(p - 1, lbig - 1), down_to = std::min(p, lbig - 1);
  if (up_from >= 1 || down_to >= 1) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t need = std::max<int64_t>(1, (1ll << std::max(up_from, down_to)) / 2);
    dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)sweep_blocks_per_sm * sms, need)));
    hm::TreeParams arg = tp;
    int a1 = up_from, a2 = 1, a3 = 1, a4 = down_to;
    void* args[] = {&arg, &a1, &a2, &a3, &a4};
    cudaError_t e = cudaSuccess;
    st = launch("hss_tree_sweep", s, [&] {
      e = cudaLaunchCooperativeKernel((const void*)hm::hss_tree_sweep_kernel<KT, NT>, grid, dim3(256), args, smem, s);
    });
    if (st == HM_OK && e != cudaSuccess) return fail(HM_ERR_CUDA, "hss_tree_sweep: %s", cudaGetErrorString(e));
    if (st) return st;
  }
  // downsweep: big levels lbig .. p one launch each
  for (int l = std::max(lbig, 1); l <= p; ++l) {
    const unsigned pairs = (unsigned)(1ll << (l - 1));
    st = launch("hss_down_level", s, [&] { hm::hss_down_pair_kernel<KT, NT, MINB><<<pairs, 256, smem, s>>>(tp, l); });
    if (st) return st;
  }
  return HM_OK;
}

hm_status tree_dispatch(const hm::TreeParams& tp, int p, int k, int nt, cudaStream_t s) {
#define HM_TREE(KT_)                                           \
  if (k == KT_) {                                              \
    if (nt == 1) return tree_launch<KT_, 1>(tp, p, s);         \
    if (nt == 2) return tree_launch<KT_, 2>(tp, p, s);         \
    return tree_launch<KT_, 4>(tp, p, s);                      \
  }
  HM_TREE(16)
  HM_TREE(32)
  HM_TREE(64)
#undef HM_TREE
  return fail(HM_ERR_UNSUPPORTED, "hss tree: no instance for k=%d", k);
}

hm_status hss_run(const hm_tree* tree, int32_t k, const double* D, const double* U, const double* V,
                  const double* R, const double* W, const double* B, const double* X, int32_t nrhs, double* Y,
                  void* ws, size_t ws_bytes, cudaStream_t stream, int32_t flags) {
  HssPlan P;
  hm_status st = hss_plan(tree, k, nrhs, flags, &P);
  if (st) return st;
  if (!ws || ws_bytes < P.total) return fail(HM_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, P.total);
  if (!D || !X || !Y) return fail(HM_ERR_INVALID_ARG, "NULL D / X / Y pointer");
  if (k > 0 && P.p > 0 && (!U || !V || !B)) return fail(HM_ERR_INVALID_ARG, "NULL U / V / B pointer");
  if (k > 0 && P.p > 1 && (!R || !W)) return fail(HM_ERR_INVALID_ARG, "NULL R / W pointer");
  if (!aligned16(D) || !aligned16(ws)) return fail(HM_ERR_INVALID_ARG, "D and workspace must be 16-byte aligned");
  if (k > 0 && P.p > 0 && (!aligned16(U) || !aligned16(V) || !aligned16(B) || (P.p > 1 && (!aligned16(R) || !aligned16(W)))))
    return fail(HM_ERR_INVALID_ARG, "U, V, R, W, B must be 16-byte aligned");
  const size_t xy_bytes = sizeof(double) * (size_t)(P.n * nrhs);
  if (overlap(X, xy_bytes, Y, xy_bytes)) return fail(HM_ERR_INVALID_ARG, "X and Y overlap");
  if (!(flags & HM_WS_HOSTIO) && (!aligned16(X) || !aligned16(Y)))
    return fail(HM_ERR_INVALID_ARG, "X and Y must be 16-byte aligned");

  char* w = static_cast<char*>(ws);
  double* xh = reinterpret_cast<double*>(w + P.off_xh);
  double* yh = reinterpret_cast<double*>(w + P.off_yh);
  const double* Xd = X;
  double* Yd = Y;
  g_launches = 0;
  prof_new_call();
  if (flags & HM_WS_HOSTIO) {
    Xd = reinterpret_cast<double*>(w + P.off_x);
    Yd = reinterpret_cast<double*>(w + P.off_y);
    if (cudaMemcpyAsync(const_cast<double*>(Xd), X, xy_bytes, cudaMemcpyHostToDevice, stream) != cudaSuccess)
      return cuda_check("H2D copy of X");
  }
  const int64_t km = (int64_t)k * nrhs;
  const bool coupled = (k > 0 && P.p > 0);
  if (coupled) {
    // Step 1: v_i^p = V_i^T X(I_i) for every leaf (node size b: always complete)
    double* xleaf = xh + (((int64_t)1 << P.p) - 2) * km;
    if (P.vt == VtPath::kMma) {
      hm::BatchedVtParams bp{V, P.b * k, Xd, P.b * nrhs, xleaf, km, (int64_t)1 << P.p, (int32_t)P.b, nrhs};
      if ((st = vt_batched_dispatch("vt_contract", bp, k, P.nt_vt, stream))) return st;
    } else {
      hm::VtParams vp;
      memset(&vp, 0, sizeof vp);
      vp.X = Xd; vp.n = P.n; vp.m = nrhs; vp.mc = P.mc_vt; vp.tile = P.tile; vp.nlev = 1;
      vp.lev[0].V = V; vp.lev[0].k = k; vp.lev[0].s = P.b;
      vp.lev[0].out = xleaf;
      vp.lev[0].partial = nullptr;
      st = (P.vt == VtPath::kGemv) ? vt_gemv_dispatch(vp, P.b, k, stream) : vt_generic(vp, P.n, stream);
      if (st) return st;
    }
    if (P.mma_levels) {
      // Step 1 (cont.) upsweep + Steps 2-3 coupling/downsweep: one cooperative launch
      hm::TreeParams tp{W, R, B, xh, yh, nrhs, 0, 0, 0};
      if ((st = tree_dispatch(tp, P.p, k, P.nt_down, stream))) return st;
    } else {
      // Step 1 (cont.): upsweep l = p-1 .. 1 through W^T
      for (int l = P.p - 1; l >= 1; --l) {
        hm::HssLevelParams hp{W, B, xh, yh, l, k, nrhs, 0};
        const int64_t total = ((int64_t)1 << l) * km;
        const unsigned blocks = (unsigned)std::min<int64_t>((total + hm::kThreads - 1) / hm::kThreads, 148 * 16);
        st = launch("hss_up_level", stream,
                    [&] { hm::hss_up_level_kernel<<<blocks, hm::kThreads, 0, stream>>>(hp); });
        if (st) return st;
      }
      // Steps 2+3: coupling on level l (cores of the parents) + downsweep from l-1
      for (int l = 1; l <= P.p; ++l) {
        hm::HssLevelParams hp{R, B, xh, yh, l, k, nrhs, 0};
        const int64_t total = ((int64_t)1 << l) * km;
        const unsigned blocks = (unsigned)std::min<int64_t>((total + hm::kThreads - 1) / hm::kThreads, 148 * 16);
        st = launch("hss_down_level", stream,
                    [&] { hm::hss_down_level_kernel<<<blocks, hm::kThreads, 0, stream>>>(hp); });
        if (st) return st;
      }
    }
  }
  // Step 4: Y(I_i) = U_i y_i^p + D_i X(I_i)
  hm::LeafParams lp;
  memset(&lp, 0, sizeof lp);
  lp.D = D; lp.X = Xd; lp.Y = Yd; lp.b = P.b; lp.m = nrhs; lp.mc = P.mc_leaf;
  if (coupled) {
    hm::LeafSeg& sg = lp.seg[lp.nseg++];
    sg.A = U;
    sg.T = yh + (((int64_t)1 << P.p) - 2) * km;
    sg.k = k; sg.shift = 0; sg.xr = 0;
    lp.ktot = k;
  }
  if ((st = leaf_dispatch(lp, 1ll << P.p, P.leaf, coupled ? k : 0, P.nt_leaf, P.mc_leaf, stream))) return st;
  if (flags & HM_WS_HOSTIO) {
    if (cudaMemcpyAsync(Y, Yd, xy_bytes, cudaMemcpyDeviceToHost, stream) != cudaSuccess)
      return cuda_check("D2H copy of Y");
  }
  return HM_OK;
}

}  // namespace

extern "C" {

hm_status hm_hodlr_workspace_bytes(const hm_tree* tree, const int32_t* ranks, int32_t nrhs, int32_t flags,
                                   size_t* bytes) {
  if (!bytes) return fail(HM_ERR_INVALID_ARG, "bytes is NULL");
  HodlrPlan P;
  hm_status st = hodlr_plan(tree, ranks, nrhs, flags, &P);
  if (st) return st;
  *bytes = P.total;
  return HM_OK;
}

hm_status hodlr_matvec(const hm_tree* tree, const int32_t* ranks, const double* D, const double* U,
                       const double* V, const double* X, int32_t nrhs, double* Y, void* workspace,
                       size_t workspace_bytes, void* stream) {
  return hodlr_run(tree, ranks, D, U, V, X, nrhs, Y, workspace, workspace_bytes,
                   static_cast<cudaStream_t>(stream), 0);
}

hm_status hodlr_matvec_hostio(const hm_tree* tree, const int32_t* ranks, const double* D, const double* U,
                              const double* V, const double* X_host, int32_t nrhs, double* Y_host,
                              void* workspace, size_t workspace_bytes, void* stream) {
  return hodlr_run(tree, ranks, D, U, V, X_host, nrhs, Y_host, workspace, workspace_bytes,
                   static_cast<cudaStream_t>(stream), HM_WS_HOSTIO);
}

hm_status hm_hss_workspace_bytes(const hm_tree* tree, int32_t k, int32_t nrhs, int32_t flags, size_t* bytes) {
  if (!bytes) return fail(HM_ERR_INVALID_ARG, "bytes is NULL");
  HssPlan P;
  hm_status st = hss_plan(tree, k, nrhs, flags, &P);
  if (st) return st;
  *bytes = P.total;
  return HM_OK;
}

hm_status hss_matvec(const hm_tree* tree, int32_t k, const double* D, const double* U, const double* V,
                     const double* R, const double* W, const double* B, const double* X, int32_t nrhs,
                     double* Y, void* workspace, size_t workspace_bytes, void* stream) {
  return hss_run(tree, k, D, U, V, R, W, B, X, nrhs, Y, workspace, workspace_bytes,
                 static_cast<cudaStream_t>(stream), 0);
}

hm_status hss_matvec_hostio(const hm_tree* tree, int32_t k, const double* D, const double* U, const double* V,
                            const double* R, const double* W, const double* B, const double* X_host,
                            int32_t nrhs, double* Y_host, void* workspace, size_t workspace_bytes, void* stream) {
  return hss_run(tree, k, D, U, V, R, W, B, X_host, nrhs, Y_host, workspace, workspace_bytes,
                 static_cast<cudaStream_t>(stream), HM_WS_HOSTIO);
}

const char* hm_last_error(void) { return g_err.c_str(); }

hm_status hm_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_on = on != 0;
  return HM_OK;
}

hm_status hm_profile_collect(hm_launch_record* out, int32_t cap, int32_t* count) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (cap > 0 && !out) return fail(HM_ERR_INVALID_ARG, "out is NULL");
  int32_t n = 0;
  hm_status st = HM_OK;
  for (const TraceRec& r : g_prof_recs) {
    if (n < cap) {
      float ms = 0.f;
      if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess)
        st = cuda_check("hm_profile_collect");
      memset(&out[n], 0, sizeof out[n]);
      strncpy(out[n].name, r.name, sizeof out[n].name - 1);
      out[n].call = r.call;
      out[n].ms = ms;
    }
    ++n;
    g_prof_pool.push_back(r.a);
    g_prof_pool.push_back(r.b);
  }
  g_prof_recs.clear();
  g_prof_call = -1;
  if (count) *count = n;
  return st;
}
int32_t hm_abi_version(void) { return HM_ABI_VERSION; }
int32_t hm_last_launch_count(void) { return g_launches; }

}  // extern "C"
