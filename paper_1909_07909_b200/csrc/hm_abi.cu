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
#include "hm_vec.cuh"
#include "hm_convert.cuh"
#include "hm_general.cuh"
#include "hm_leafup.cuh"
#include "hm_small.cuh"
#include "hm_treegemv.cuh"

// One-launch HODLR for small problems (hodlr_small_kernel): correct (parity
// tested with HM_SMALL_HODLR=1) but not faster on config 1 (22.9 vs 21 us per
// call: the kernel alone takes 17.7 us, the two-kernel path 20.5 us of device
// time); off by default (r01_tuning.md).
#ifndef HM_VT_LV_MIN_M
#define HM_VT_LV_MIN_M 17  // X re-reads of vt_mma_levels fall out of L2 above this (config 3, m = 64)
#endif
#ifndef HM_VT_TILE4
#define HM_VT_TILE4 1  // vt_mma_levels on 4-leaf tiles below the vt_lv threshold
#endif
#ifndef HM_SMALL_HODLR
#define HM_SMALL_HODLR 0
#endif
#define HM_NO_SMALL_HODLR (!HM_SMALL_HODLR)

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
#ifndef HM_VT16_NTMAX
#define HM_VT16_NTMAX 8
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
//
// A HODLR problem is planned on a row block of n rows that is a whole subtree
// of depth p (leaf b), plus q "top" levels whose nodes contain the whole block
// (q > 0 only for one rank of the distributed product). Levels
// keep their global index: top levels 1..q, subtree levels q+1..q+p;
// ranks[l-1] = k_l for all of them.

enum class VtPath { kNone, kGeneric, kGemv, kMma };
enum class LeafPath { kGeneric, kGemv, kMma };  // kGemv: TMA ring when the shape allows (leaf_gemv_tma)

struct HodlrPlan {
  int64_t n, b;
  int32_t p, q, m, k;  // k = the common nonzero rank (0 if all zero); the largest one when kvary
  bool kvary;          // per-level ranks on the uniform tree: levels grouped by rank
  int64_t ktot;        // sum over all q + p levels
  int64_t top_doubles; // sum_{l <= q} k_l m (the distributed exchange block)
  VtPath vt;
  LeafPath leaf;
  int32_t mc_vt, mc_leaf, nt_vt, nt_leaf;
  int64_t tile;  // rows per vt CTA
  size_t off_t[hm::kMaxLevels + 1];
  size_t off_part[hm::kMaxLevels + 1];
  size_t off_ttop, off_spart, off_x, off_y, total;
};

// Column tiles (of 8) per V^T X pass of vt_mma_levels: as many as the
// accumulators allow, so V is streamed once per pass (k <= 16: up to 64
// columns, NT = 8; measured on config 3 at m = 64: 1769 -> 1403 us for k = 16).
int vt_mma_nt(int k, int nrhs) { return nt_for(nrhs, k == 64 ? 2 : (k == 32 ? 4 : (k == 16 ? HM_VT16_NTMAX : 8))); }

hm_status hodlr_plan_ex(int64_t n, int64_t b, int32_t p, int32_t q, const int32_t* ranks, int32_t nrhs,
                        int32_t flags, HodlrPlan* P, bool allow_vary = false) {
  if (nrhs < 1) return fail(HM_ERR_INVALID_ARG, "nrhs = %d < 1", nrhs);
  if (p + q > 0 && !ranks) return fail(HM_ERR_INVALID_ARG, "ranks is NULL");
  if (p + q + 1 > hm::kMaxLevels) return fail(HM_ERR_UNSUPPORTED, "too many levels");
  memset(P, 0, sizeof *P);
  P->n = n; P->b = b; P->p = p; P->q = q; P->m = nrhs;
  for (int l = 1; l <= p + q; ++l) {
    const int k = ranks[l - 1];
    if (k < 0) return fail(HM_ERR_INVALID_ARG, "ranks[%d] = %d < 0", l - 1, k);
    if (k > hm::kMaxRank) return fail(HM_ERR_UNSUPPORTED, "rank %d > %d", k, hm::kMaxRank);
    if (k > 0) {
      if (P->k != 0 && P->k != k) {
        if (!allow_vary)
          return fail(HM_ERR_UNSUPPORTED, "per-level ranks differ (%d vs %d); variable ranks (P:264) not built here",
                      P->k, k);
        P->kvary = true;
      }
      P->k = std::max(P->k, k);
    }
    P->ktot += k;
    if (l <= q) P->top_doubles += (int64_t)k * nrhs;
  }
  const int64_t k = P->k;
  const bool tiles8 = p >= 3;  // 8-leaf row tiles exist
  if (P->kvary) {
    // Per-level ranks on the uniform tree, 8-leaf row tiles: one V^T X
    // pass per distinct rank — the tuned kernel where the rank fits it (GEMV:
    // powers of two <= 64 at nrhs = 1; DMMA: 16/32/64 at nrhs >= 2), else
    // vt_contract on the same tiles — and ONE leaf pass with per-segment ranks.
    // Other shapes (p < 3, leaf not a multiple of 64) take the general-tree kernels.
    if (!(tiles8 && b % 64 == 0 && b <= 1024))
      return fail(HM_ERR_UNSUPPORTED, "per-level ranks: uniform-tree kernels need levels >= 3 and leaf %% 64 == 0");
    P->vt = nrhs == 1 ? VtPath::kGemv : VtPath::kMma;
    P->tile = (nrhs >= 2 && HM_VT_TILE4 && nrhs < HM_VT_LV_MIN_M) ? 4 * b : 8 * b;
    int mc = std::min<int32_t>(nrhs, hm::kMaxMc);
    while (mc > 1 && P->tile * mc + hm::kThreads > kSmemBudgetDoubles) --mc;
    P->mc_vt = mc;
    bool pow2 = true, k8 = true;
    for (int l = 1; l <= p + q; ++l) {
      const int kl = ranks[l - 1];
      if (kl == 0) continue;
      pow2 = pow2 && pow2_rank(kl, 1, 64);
      k8 = k8 && kl % 8 == 0;
    }
    P->leaf = LeafPath::kGeneric;
    if (nrhs == 1 && pow2 && (2 * b + (int64_t)(p + q) * k) * 8 <= 160 * 1024) {
      P->leaf = LeafPath::kGemv;
    } else if (nrhs >= 2 && (b == 64 || b == 128 || b == 256) && k8) {
      const int rg = (int)(b / 64);
      P->nt_leaf = nt_for(nrhs, rg == 4 ? 2 : 4);
      if ((b + P->ktot) * (8 * P->nt_leaf + 4) <= kSmemBudgetDoubles) P->leaf = LeafPath::kMma;
    }
  } else {
  if (k == 0 || p + q == 0) {
    P->vt = VtPath::kNone;
  } else if (nrhs == 1 && tiles8 && b % 64 == 0 && b <= 4096 && pow2_rank((int)k, 1, 64)) {
    P->vt = VtPath::kGemv;
    P->tile = 8 * b;
  } else if (nrhs >= 2 && tiles8 && b % 4 == 0 && pow2_rank((int)k, 1, 64)) {
    P->vt = VtPath::kMma;
    P->tile = (HM_VT_TILE4 && nrhs < HM_VT_LV_MIN_M) ? 4 * b : 8 * b;  // vt_lv (m >= HM_VT_LV_MIN_M) needs 8
    P->nt_vt = vt_mma_nt((int)k, nrhs);
  } else {
    P->vt = VtPath::kGeneric;
    P->mc_vt = vt_mc(b, nrhs);
    P->tile = pick_tile(b, p, P->mc_vt);
  }
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
  }
  if (P->leaf == LeafPath::kGeneric) {
    P->mc_leaf = pick_mc(b, P->ktot, nrhs);
    if ((b + P->ktot) * P->mc_leaf > kSmemBudgetDoubles)
      return fail(HM_ERR_UNSUPPORTED, "leaf %lld + ranks %lld too large for shared-memory staging", (long long)b,
                  (long long)P->ktot);
  }
  // workspace: subtree t_l, per-tile partials where a node spans several tiles
  // (every top level: its node is the whole block), combined top t blocks
  size_t off = 0;
  for (int l = q + 1; l <= q + p; ++l) {
    P->off_t[l] = off;
    off = align_up(off + sizeof(double) * (size_t)((1ll << (l - q)) * ranks[l - 1] * nrhs));
  }
  for (int l = 1; l <= q + p; ++l) {
    const int64_t s = l <= q ? n : (n >> (l - q));
    P->off_part[l] = off;
    if (P->vt != VtPath::kNone && ranks[l - 1] > 0 && s > P->tile)
      off = align_up(off + sizeof(double) * (size_t)((n / P->tile) * ranks[l - 1] * nrhs));
  }
  P->off_ttop = off;
  off = align_up(off + sizeof(double) * (size_t)P->top_doubles);
  // small problems (hodlr_small_kernel, HM_SMALL_HODLR): per-leaf partials
  P->off_spart = off;
  if (HM_SMALL_HODLR) off = align_up(off + sizeof(double) * (size_t)(((int64_t)1 << p) * P->ktot * nrhs));
  P->off_x = P->off_y = off;
  if (flags & HM_WS_HOSTIO) {
    P->off_x = off;
    off = align_up(off + sizeof(double) * (size_t)(n * nrhs));
    P->off_y = off;
    off = align_up(off + sizeof(double) * (size_t)(n * nrhs));
  }
  P->total = std::max<size_t>(off, kAlign);
  return HM_OK;
}

hm_status hodlr_plan(const hm_tree* tree, const int32_t* ranks, int32_t nrhs, int32_t flags, HodlrPlan* P) {
  hm_status st = check_tree(tree);
  if (st) return st;
  return hodlr_plan_ex(tree->n, tree->leaf, tree->levels, 0, ranks, nrhs, flags, P, /*allow_vary=*/true);
}

// ---- leaf launches (shared by HODLR and HSS) ----

template <int MC>
hm_status launch_leaf_generic(const hm::LeafParams& lp, int64_t nleaves, cudaStream_t s) {
  size_t smem = sizeof(double) * (size_t)((lp.b + lp.ktot) * MC);
  allow_smem(hm::leaf_apply_kernel<MC>, smem);
  dim3 grid((unsigned)nleaves, (unsigned)((lp.m + MC - 1) / MC));
  return launch(lp.dtrans ? "leaf_apply_t" : "leaf_apply", s,
                [&] { hm::leaf_apply_kernel<MC><<<grid, hm::kThreads, smem, s>>>(lp); });
}

template <int K, int NCH, bool VARK = false>
hm_status launch_leaf_gemv_n(const hm::LeafParams& lp, int64_t nleaves, cudaStream_t s) {
  constexpr int ROWS = NCH >= 8 ? 2 : (NCH == 0 ? 4 : HM_GEMV_ROWS);
  if (lp.dtrans) {  // adjoint: D_i^T x_i, per-warp column partials in shared memory
    const size_t smem = sizeof(double) * (size_t)(10 * lp.b + lp.nseg * K);
    allow_smem(hm::leaf_gemv_kernel<K, NCH, ROWS, true, VARK>, smem);
    return launch("leaf_gemv_t", s,
                  [&] { hm::leaf_gemv_kernel<K, NCH, ROWS, true, VARK><<<(unsigned)nleaves, 256, smem, s>>>(lp); });
  }
  size_t smem = sizeof(double) * (size_t)(2 * lp.b + lp.nseg * K);
  allow_smem(hm::leaf_gemv_kernel<K, NCH, ROWS, false, VARK>, smem);
  return launch("leaf_gemv", s,
                [&] { hm::leaf_gemv_kernel<K, NCH, ROWS, false, VARK><<<(unsigned)nleaves, 256, smem, s>>>(lp); });
}

#ifndef HM_NO_TMA
#define HM_NO_TMA 0
#endif
constexpr int kTmaStages = 6;

template <int K, int NCH>
hm_status launch_leaf_gemv_tma(const hm::LeafParams& lp, int64_t nleaves, cudaStream_t s) {
  const size_t smem = (size_t)kTmaStages * hm::kTmaChunkBytes + 2 * kTmaStages * sizeof(uint64_t) +
                      sizeof(double) * (size_t)(2 * 64 * NCH + lp.nseg * K);
  allow_smem(hm::leaf_gemv_tma_kernel<K, NCH>, smem);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)std::min<int64_t>(nleaves, sms);
  return launch("leaf_gemv_tma", s, [&] {
    hm::leaf_gemv_tma_kernel<K, NCH><<<grid, 32 * (hm::kTmaConsumers + 1), smem, s>>>(lp, nleaves, kTmaStages);
  });
}

// nrhs = 1 leaf pass, measured (r01_tuning.md): the TMA ring wins for k >= 8
// at b = 256 (config 3 m=1: 594 vs 631 us) and b = 64 (config 1: 20 vs 29 us
// per call); the register-streaming kernel wins for k < 8 (config 5: 5.25 vs
// 6.45 ms) and at b = 128 (config 4 at m=1, k=32: 830 vs 1041 us).
template <int K>
hm_status launch_leaf_gemv(const hm::LeafParams& lp, int64_t nleaves, cudaStream_t s) {
  if constexpr (K >= 8 && K <= 32) {
    if (!HM_NO_TMA && !lp.dtrans && lp.b != 128 && lp.b * K <= 4096) {
      switch (lp.b) {
        case 64: return launch_leaf_gemv_tma<K, 1>(lp, nleaves, s);
        case 128: return launch_leaf_gemv_tma<K, 2>(lp, nleaves, s);
        case 256: return launch_leaf_gemv_tma<K, 4>(lp, nleaves, s);
        case 512: if constexpr (K <= 8) return launch_leaf_gemv_tma<K, 8>(lp, nleaves, s); break;
        default: break;
      }
    }
  }
  switch (lp.b) {
    case 64: return launch_leaf_gemv_n<K, 1>(lp, nleaves, s);
    case 128: return launch_leaf_gemv_n<K, 2>(lp, nleaves, s);
    case 256: return launch_leaf_gemv_n<K, 4>(lp, nleaves, s);
    case 512: return launch_leaf_gemv_n<K, 8>(lp, nleaves, s);
    default: return launch_leaf_gemv_n<K, 0>(lp, nleaves, s);
  }
}

// (RG, NT) -> prefetch depth and launch-bound occupancy (measured, r01_tuning.md)
template <int RG, int NT>
struct LeafMmaTune {
#ifdef HM_LEAF_PF_OVR  // development overrides (tools/kbench.py A/B builds)
  static constexpr int PF = HM_LEAF_PF_OVR;
#else
  static constexpr int PF = (RG == 2 && NT == 4) ? 1 : 2;
#endif
#ifdef HM_LEAF_MINB_OVR
  static constexpr int MINB = HM_LEAF_MINB_OVR;
#else
  static constexpr int MINB = (RG == 2 && NT == 4) ? 4 : 0;
#endif
};

template <int RG, int NT>
hm_status launch_leaf_mma(const hm::LeafParams& lp, int64_t nleaves, cudaStream_t s) {
  constexpr int PF = LeafMmaTune<RG, NT>::PF, MINB = LeafMmaTune<RG, NT>::MINB;
  size_t smem = sizeof(double) * (size_t)((lp.b + lp.ktot) * (NT * 8 + 4));
  const int64_t chunks = (lp.m + NT * 8 - 1) / (NT * 8);
  if (lp.dp > 0) {  // HSS: leaf-level coupling + downsweep fused (y_i computed in the CTA)
    const size_t sm2 = smem + sizeof(double) * 2 * (size_t)lp.seg[0].k * (NT * 8 + 2);
    allow_smem(hm::leaf_mma_kernel<RG, NT, PF, MINB, false, true>, sm2);
    return launch("leaf_mma_down", s, [&] {
      hm::leaf_mma_kernel<RG, NT, PF, MINB, false, true><<<(unsigned)(nleaves * chunks), 256, sm2, s>>>(lp);
    });
  }
  if (lp.dtrans) {
    allow_smem(hm::leaf_mma_kernel<RG, NT, PF, MINB, true>, smem);
    return launch("leaf_mma_t", s, [&] {
      hm::leaf_mma_kernel<RG, NT, PF, MINB, true><<<(unsigned)(nleaves * chunks), 256, smem, s>>>(lp);
    });
  }
  allow_smem(hm::leaf_mma_kernel<RG, NT, PF, MINB>, smem);
  return launch("leaf_mma", s, [&] {
    hm::leaf_mma_kernel<RG, NT, PF, MINB><<<(unsigned)(nleaves * chunks), 256, smem, s>>>(lp);
  });
}

hm_status leaf_dispatch(const hm::LeafParams& lp, int64_t nleaves, LeafPath path, int k, int nt, int mc,
                        cudaStream_t s, bool kvary = false) {
  if (path == LeafPath::kGemv && kvary) {  // per-level ranks: k = the largest (register streaming kernel)
#define HM_LEAF_VARK(K_)                                          \
  if (k == K_) switch (lp.b) {                                    \
      case 64: return launch_leaf_gemv_n<K_, 1, true>(lp, nleaves, s);  \
      case 128: return launch_leaf_gemv_n<K_, 2, true>(lp, nleaves, s); \
      case 256: return launch_leaf_gemv_n<K_, 4, true>(lp, nleaves, s); \
      default: break;                                             \
    }
    HM_LEAF_VARK(2)
    HM_LEAF_VARK(4)
    HM_LEAF_VARK(8)
    HM_LEAF_VARK(16)
    HM_LEAF_VARK(32)
    HM_LEAF_VARK(64)
#undef HM_LEAF_VARK
    return fail(HM_ERR_UNSUPPORTED, "leaf_gemv (per-level ranks): no instance for k=%d b=%lld", k, (long long)lp.b);
  }
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
  return launch("vt_gemv", s,
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

// vp.tile = LPC b rows per CTA: 4 leaves when the plan chose it (m below the
// vt_lv threshold: twice the CTAs, so the grid fills every SM evenly), else 8
template <int KT, int NT>
hm_status vt_mma_launch(const hm::VtParams& vp, int64_t b, cudaStream_t s) {
  if (vp.tile == 4 * b) {
    size_t smem = sizeof(double) * (size_t)(4 * KT * NT * 8);
    allow_smem(hm::vt_mma_levels_kernel<KT, NT, 4>, smem);
    return launch("vt_mma_levels", s, [&] {
      hm::vt_mma_levels_kernel<KT, NT, 4><<<(unsigned)(vp.n / (4 * b)), 128, smem, s>>>(vp, b);
    });
  }
  size_t smem = sizeof(double) * (size_t)(8 * KT * NT * 8);
  allow_smem(hm::vt_mma_levels_kernel<KT, NT>, smem);
  return launch("vt_mma_levels", s, [&] {
    hm::vt_mma_levels_kernel<KT, NT><<<(unsigned)(vp.n / (8 * b)), 256, smem, s>>>(vp, b);
  });
}

hm_status vt_mma_dispatch(const hm::VtParams& vp, int64_t b, int k, int nt, cudaStream_t s) {
#define HM_VT_MMA(KT_)                                                         \
  if (k == KT_) {                                                              \
    if (nt == 1) return vt_mma_launch<KT_, 1>(vp, b, s);                       \
    if (nt == 2) return vt_mma_launch<KT_, 2>(vp, b, s);                       \
    if constexpr (KT_ == 16) if (nt == 8) return vt_mma_launch<KT_, 8>(vp, b, s); \
    if constexpr (KT_ < 64) return vt_mma_launch<KT_, 4>(vp, b, s);             \
  }
  HM_VT_MMA(16)
  HM_VT_MMA(32)
  HM_VT_MMA(64)
#undef HM_VT_MMA
#define HM_VT_MMA_SMALL(KT_)                                                   \
  if (k == KT_) {                                                              \
    if (nt == 1) return vt_mma_launch<KT_, 1>(vp, b, s);                       \
    if (nt == 2) return vt_mma_launch<KT_, 2>(vp, b, s);                       \
    if (nt == 4) return vt_mma_launch<KT_, 4>(vp, b, s);                       \
    return vt_mma_launch<KT_, 8>(vp, b, s);                                    \
  }
  HM_VT_MMA_SMALL(1)
  HM_VT_MMA_SMALL(2)
  HM_VT_MMA_SMALL(4)
  HM_VT_MMA_SMALL(8)
#undef HM_VT_MMA_SMALL
  return fail(HM_ERR_UNSUPPORTED, "vt_mma: no instance for k=%d nt=%d", k, nt);
}

// Many right-hand sides: the level-parallel pipelined kernel (vt_lv_kernel, X
// and V read once). Returns HM_ERR_UNSUPPORTED when the shape does not fit it.
#ifndef HM_VT_LV_NW
#define HM_VT_LV_NW 16
#endif
#ifndef HM_VT_LV_NT
#define HM_VT_LV_NT 2
#endif
#ifndef HM_VT_LV_R
#define HM_VT_LV_R 32  // rows per pipeline stage (measured: 8 / 16 / 32 -> 1216 / 1107 / 1033 us, config 3 m=64)
#endif
template <int KT, int IPW, int NS>
hm_status vt_lv_launch(const hm::VtParams& vp, int64_t b, size_t smem, cudaStream_t s) {
  constexpr int NW = HM_VT_LV_NW, NT = HM_VT_LV_NT;
  allow_smem(hm::vt_lv_kernel<KT, NT, IPW, HM_VT_LV_R, NS, NW>, smem);
  return launch("vt_lv", s, [&] {
    hm::vt_lv_kernel<KT, NT, IPW, HM_VT_LV_R, NS, NW><<<(unsigned)(vp.n / (8 * b)), NW * 32, smem, s>>>(vp, b);
  });
}

hm_status vt_lv_dispatch(const hm::VtParams& vp, int64_t b, int k, cudaStream_t s) {
  constexpr int R = HM_VT_LV_R, NW = HM_VT_LV_NW, MC = 8 * HM_VT_LV_NT;
  if (HM_VT_LV_MIN_M <= 0 || vp.m < HM_VT_LV_MIN_M || !(k == 16 || k == 32) || b % R != 0 || vp.nlev < 1)
    return HM_ERR_UNSUPPORTED;
  const int mp = (vp.m + MC - 1) / MC * MC;
  const int items = vp.nlev * (k / 16) * (mp / MC);
  const int ipw = (items + NW - 1) / NW;
  if (ipw > 4) return HM_ERR_UNSUPPORTED;
  const int64_t sd = hm::vt_lv_stage_doubles(R, k, vp.nlev, mp);
  int ns = 0;
  if (4 * sd * 8 <= 220 * 1024) ns = 4;
  else if (2 * sd * 8 <= 220 * 1024) ns = 2;
  if (!ns) return HM_ERR_UNSUPPORTED;
  const size_t smem = (size_t)ns * sd * 8;
#define HM_LV(KT_, IPW_)                                                               \
  if (k == KT_ && ipw == IPW_)                                                         \
    return ns == 4 ? vt_lv_launch<KT_, IPW_, 4>(vp, b, smem, s) : vt_lv_launch<KT_, IPW_, 2>(vp, b, smem, s);
  HM_LV(16, 1) HM_LV(16, 2) HM_LV(16, 3) HM_LV(16, 4)
  HM_LV(32, 1) HM_LV(32, 2) HM_LV(32, 3) HM_LV(32, 4)
#undef HM_LV
  return HM_ERR_UNSUPPORTED;
}

hm_status vt_mma_any(const hm::VtParams& vp, int64_t b, int k, int nt, cudaStream_t s) {
  const hm_status st = vt_lv_dispatch(vp, b, k, s);
  if (st != HM_ERR_UNSUPPORTED) return st;
  return vt_mma_dispatch(vp, b, k, nt, s);
}

template <int KT, int NT>
#ifndef HM_VTB_MPW
#define HM_VTB_MPW 2  // 32 rank columns per warp when k allows (measured, r01_tuning.md)
#endif
hm_status vt_batched_launch(const char* name, const hm::BatchedVtParams& bp, cudaStream_t s) {
  constexpr int MPW = (KT / 16) % HM_VTB_MPW == 0 ? HM_VTB_MPW : 1;
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

// Phase 1 of the HODLR product: V_l^T X for the levels [l0, l1] (global
// indices) in one pass over row tiles, per-tile partials -> fixed-order reduce.
// Top levels (l <= q) have one node = the whole block; their result goes to
// `top_out` (packed [sum_{l<=q} k_l][m]); subtree levels go to the workspace.
hm_status hodlr_vt_phase(const HodlrPlan& P, const int32_t* ranks, const double* V, const double* Xd, char* w,
                         int l0, int l1, double* top_out, cudaStream_t stream) {
  if (P.vt == VtPath::kNone) return HM_OK;
  const int nrhs = P.m;
  hm::VtParams vp;
  memset(&vp, 0, sizeof vp);
  vp.X = Xd; vp.n = P.n; vp.m = nrhs; vp.mc = P.mc_vt; vp.tile = P.tile;
  hm::ReduceParams rp;
  memset(&rp, 0, sizeof rp);
  int64_t uoff = 0, toff = 0;
  for (int l = 1; l <= P.q + P.p; ++l) {
    const int k = ranks[l - 1];
    const int64_t s = l <= P.q ? P.n : (P.n >> (l - P.q));
    if (k > 0 && l >= l0 && l <= l1) {
      hm::VtLevel& lv = vp.lev[vp.nlev++];
      lv.V = V + uoff;
      lv.k = k;
      lv.s = s;
      lv.out = l <= P.q ? top_out + toff : reinterpret_cast<double*>(w + P.off_t[l]);
      lv.partial = reinterpret_cast<double*>(w + P.off_part[l]);
      if (s > P.tile) {
        hm::ReduceLevel& rl = rp.lev[rp.nlev++];
        rl.partial = lv.partial;
        rl.out = lv.out;
        rl.nodes = P.n / s;
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
    if (l <= P.q) toff += (int64_t)k * nrhs;
  }
  if (vp.nlev == 0) return HM_OK;
  hm_status st = HM_OK;
  if (P.kvary) {
    // per-level ranks: one pass per distinct rank over the levels of that rank
    // (X, small next to V, is re-read once per pass)
    for (int g = 0; g < vp.nlev; ++g) {
      const int kg = vp.lev[g].k;
      bool seen = false;
      for (int h = 0; h < g; ++h) seen = seen || vp.lev[h].k == kg;
      if (seen) continue;
      hm::VtParams vg = vp;
      vg.nlev = 0;
      for (int h = 0; h < vp.nlev; ++h)
        if (vp.lev[h].k == kg) vg.lev[vg.nlev++] = vp.lev[h];
      if (nrhs == 1 && pow2_rank(kg, 1, 64)) st = vt_gemv_dispatch(vg, P.b, kg, stream);
      else if (nrhs >= 2 && pow2_rank(kg, 1, 64))
        st = vt_mma_any(vg, P.b, kg, vt_mma_nt(kg, nrhs), stream);
      else st = vt_generic(vg, P.n, stream);  // same 8-leaf tiles (P.tile), P.mc_vt columns
      if (st) return st;
    }
  } else if (P.vt == VtPath::kGemv) st = vt_gemv_dispatch(vp, P.b, P.k, stream);
  else if (P.vt == VtPath::kMma) st = vt_mma_any(vp, P.b, P.k, P.nt_vt, stream);
  else st = vt_generic(vp, P.n, stream);
  if (st) return st;
  if (rp.nlev > 0) {
    const unsigned grid = (unsigned)((rp.threads + hm::kThreads - 1) / hm::kThreads);
    st = launch("reduce_partials", stream,
                [&] { hm::reduce_partials_kernel<<<grid, hm::kThreads, 0, stream>>>(rp); });
    if (st) return st;
  }
  return HM_OK;
}

// Phase 2: per leaf Y(I_i) = D_i X(I_i) + sum_l U_l(I_i) t_{l, sib(node_l(i))};
// for top levels the coefficient block is the same for every leaf (ttop).
hm_status hodlr_leaf_phase(const HodlrPlan& P, const int32_t* ranks, const double* D, const double* U,
                           const double* Xd, double* Yd, char* w, const double* ttop, cudaStream_t stream,
                           bool dtrans = false) {
  hm::LeafParams lp;
  memset(&lp, 0, sizeof lp);
  lp.D = D; lp.X = Xd; lp.Y = Yd; lp.b = P.b; lp.m = P.m; lp.mc = P.mc_leaf; lp.dtrans = dtrans ? 1 : 0;
  int64_t uoff = 0, toff = 0;
  for (int l = 1; l <= P.q + P.p; ++l) {
    const int k = ranks[l - 1];
    if (k > 0) {
      hm::LeafSeg& sg = lp.seg[lp.nseg++];
      sg.A = U + uoff;
      sg.k = k;
      if (l <= P.q) {
        sg.T = ttop + toff;
        sg.shift = 62;  // node index 0 for every leaf
        sg.xr = 0;
      } else {
        sg.T = reinterpret_cast<const double*>(w + P.off_t[l]);
        sg.shift = P.q + P.p - l;  // node of leaf i at level l: i >> (depth - l)
        sg.xr = 1;                 // the sibling's coefficients: A(I_a, I_sib a) = U(I_a) V(I_sib)^T
      }
      lp.ktot += k;
    }
    uoff += P.n * k;
    if (l <= P.q) toff += (int64_t)k * P.m;
  }
  return leaf_dispatch(lp, 1ll << P.p, P.leaf, P.k, P.nt_leaf, P.mc_leaf, stream, P.kvary);
}

// ---- small problems: the whole product in one cooperative launch ----

// Latency-bound sizes only: one CTA per leaf (<= 256, co-resident), the leaf's
// inputs fit in shared memory, little arithmetic per CTA.
bool hodlr_small_ok(const HodlrPlan& P) {
  return !HM_NO_SMALL_HODLR && P.q == 0 && P.p >= 1 && P.p <= 8 && P.n <= 16384 && P.m <= 16 &&
         P.ktot * P.m * P.b <= 524288 &&
         hm::hodlr_small_smem_doubles(P.b, P.ktot, P.m) * (int64_t)sizeof(double) <= 200 * 1024;
}

hm_status hodlr_small_dispatch(const HodlrPlan& P, const int32_t* ranks, const double* D, const double* U,
                               const double* V, const double* X, double* Y, char* w, cudaStream_t s) {
  hm::SmallHodlrParams sp;
  memset(&sp, 0, sizeof sp);
  sp.D = D; sp.U = U; sp.V = V; sp.X = X; sp.Y = Y;
  sp.part = reinterpret_cast<double*>(w + P.off_spart);
  sp.n = P.n; sp.b = (int32_t)P.b; sp.p = P.p; sp.m = P.m; sp.ktot = (int32_t)P.ktot;
  int64_t ko = 0;
  for (int l = 1; l <= P.p; ++l) {
    sp.k[l - 1] = ranks[l - 1];
    sp.koff[l - 1] = ko;
    ko += ranks[l - 1];
  }
  const unsigned grid = 1u << P.p;
  const size_t smem = sizeof(double) * (size_t)hm::hodlr_small_smem_doubles(P.b, P.ktot, P.m);
  // residency check cached per shared-memory size (host latency matters at these sizes)
  static thread_local size_t last_smem = 0;
  static thread_local int64_t last_cap = 0;
  if (smem != last_smem) {
    allow_smem(hm::hodlr_small_kernel, 200 * 1024);
    int per_sm = 0, dev = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hm::hodlr_small_kernel, 256, smem) != cudaSuccess)
      return cuda_check("occupancy query (hodlr_small)");
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    last_smem = smem;
    last_cap = (int64_t)per_sm * sms;
  }
  if (last_cap < (int64_t)grid) return fail(HM_ERR_UNSUPPORTED, "hodlr_small: grid not co-resident");
  void* args[] = {&sp};
  cudaError_t e = cudaSuccess;
  hm_status st = launch("hodlr_small", s, [&] {
    e = cudaLaunchCooperativeKernel((const void*)hm::hodlr_small_kernel, dim3(grid), dim3(256), args, smem, s);
  });
  if (st == HM_OK && e != cudaSuccess) return fail(HM_ERR_CUDA, "hodlr_small: %s", cudaGetErrorString(e));
  return st;
}

hm_status hodlr_check_ptrs(const HodlrPlan& P, const double* D, const double* U, const double* V, const double* X,
                           const double* Y, void* ws, size_t ws_bytes, int32_t flags) {
  if (!ws || ws_bytes < P.total)
    return fail(HM_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, P.total);
  if (!X || !Y || (P.k > 0 && (!U || !V))) return fail(HM_ERR_INVALID_ARG, "NULL generator / X / Y pointer");
  if ((D && !aligned16(D)) || !aligned16(ws) || (P.k > 0 && (!aligned16(U) || !aligned16(V))))
    return fail(HM_ERR_INVALID_ARG, "D, U, V and the workspace must be 16-byte aligned");
  const size_t xy_bytes = sizeof(double) * (size_t)(P.n * P.m);
  if (overlap(X, xy_bytes, Y, xy_bytes)) return fail(HM_ERR_INVALID_ARG, "X and Y overlap");
  if (!(flags & HM_WS_HOSTIO) && (!aligned16(X) || !aligned16(Y)))
    return fail(HM_ERR_INVALID_ARG, "X and Y must be 16-byte aligned");
  return HM_OK;
}

// op = 0: Y = A X. op = 1: Y = A^T X: A^T is HODLR on the
// same tree with U and V exchanged and D_i transposed (A^T(I_a, I_b) =
// V_l(I_a) U_l(I_b)^T), so phase 1 contracts U^T X and the leaf pass applies
// D_i^T and the V_l rows.
hm_status hodlr_run(const hm_tree* tree, const int32_t* ranks, const double* D, const double* U,
                    const double* V, const double* X, int32_t nrhs, double* Y, void* ws, size_t ws_bytes,
                    cudaStream_t stream, int32_t flags, int op = 0) {
  HodlrPlan P;
  hm_status st = hodlr_plan(tree, ranks, nrhs, flags, &P);
  if (st) return st;
  if (!D) return fail(HM_ERR_INVALID_ARG, "NULL D pointer");
  if ((st = hodlr_check_ptrs(P, D, U, V, X, Y, ws, ws_bytes, flags))) return st;
  char* w = static_cast<char*>(ws);
  const size_t xy_bytes = sizeof(double) * (size_t)(P.n * nrhs);
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
  if (op == 0 && hodlr_small_ok(P)) {  // small problem: one cooperative launch (hm_small.cuh)
    st = hodlr_small_dispatch(P, ranks, D, U, V, Xd, Yd, w, stream);
    if (st != HM_OK && st != HM_ERR_UNSUPPORTED) return st;
    if (st == HM_OK) {
      if ((flags & HM_WS_HOSTIO) && cudaMemcpyAsync(Y, Yd, xy_bytes, cudaMemcpyDeviceToHost, stream) != cudaSuccess)
        return cuda_check("D2H copy of Y");
      return HM_OK;
    }
  }
  if ((st = hodlr_vt_phase(P, ranks, op ? U : V, Xd, w, 1, P.p, nullptr, stream))) return st;
  if ((st = hodlr_leaf_phase(P, ranks, D, op ? V : U, Xd, Yd, w, nullptr, stream, op != 0))) return st;
  if (flags & HM_WS_HOSTIO) {
    if (cudaMemcpyAsync(Y, Yd, xy_bytes, cudaMemcpyDeviceToHost, stream) != cudaSuccess)
      return cuda_check("D2H copy of Y");
  }
  return HM_OK;
}

// ---- distributed HODLR ----

struct DistPart {
  int32_t P, q, rank;
};

hm_status check_part(const hm_tree* tree, const hm_part* part, DistPart* d) {
  if (!part) return fail(HM_ERR_INVALID_ARG, "part is NULL");
  const int P = part->nranks;
  if (P < 1 || (P & (P - 1)) != 0) return fail(HM_ERR_UNSUPPORTED, "nranks = %d is not a power of two", P);
  int q = 0;
  while ((1 << q) < P) ++q;
  if (q > tree->levels) return fail(HM_ERR_UNSUPPORTED, "nranks = %d > 2^levels", P);
  if (part->rank < 0 || part->rank >= P) return fail(HM_ERR_INVALID_ARG, "rank %d not in [0, %d)", part->rank, P);
  d->P = P; d->q = q; d->rank = part->rank;
  return HM_OK;
}

hm_status hodlr_dist_plan(const hm_tree* tree, const int32_t* ranks, int32_t nrhs, const hm_part* part, int32_t flags,
                          HodlrPlan* P, DistPart* d) {
  hm_status st = check_tree(tree);
  if (st) return st;
  if ((st = check_part(tree, part, d))) return st;
  return hodlr_plan_ex(tree->n >> d->q, tree->leaf, tree->levels - d->q, d->q, ranks, nrhs, flags, P);
}

// -------------------------------------------------------------------- HSS --
//
// Planned on a subtree of depth p (leaf b) over n rows; for one rank of the
// distributed product (q > 0) the workspace also holds the replicated top tree
// (levels 1..q) and the subtree root's x / y blocks.

struct HssPlan {
  int64_t n, b;
  int32_t p, q, m, k;
  VtPath vt;
  LeafPath leaf;
  bool mma_levels;   // DMMA tree kernels
  bool gemv_levels;  // warp-per-node GEMV tree kernels (nrhs <= 4), preferred over DMMA
  int32_t mc_vt, mc_leaf, nt_vt, nt_leaf, nt_down;
  int64_t tile;
  size_t off_xh, off_yh, off_txh, off_tyh, off_x, off_y, total;
};

#ifndef HM_TREE_GEMV_MAXM
#define HM_TREE_GEMV_MAXM 1  // m = 2..4: the DMMA tree levels measured faster (C4 m=2: 490 vs 560 us)
#endif
constexpr int kTreeGemvMaxM = HM_TREE_GEMV_MAXM;

hm_status hss_plan_ex(int64_t n, int64_t b, int32_t p, int32_t q, int32_t k, int32_t nrhs, int32_t flags, HssPlan* P) {
  if (nrhs < 1) return fail(HM_ERR_INVALID_ARG, "nrhs = %d < 1", nrhs);
  if (k < 0) return fail(HM_ERR_INVALID_ARG, "k = %d < 0", k);
  if (k > hm::kMaxRank) return fail(HM_ERR_UNSUPPORTED, "rank %d > %d", k, hm::kMaxRank);
  memset(P, 0, sizeof *P);
  P->n = n; P->b = b; P->p = p; P->q = q; P->m = nrhs; P->k = k;
  const bool coupled = (k > 0 && p + q > 0);
  const bool leaf_coupled = (k > 0 && (p > 0 || q > 0));
  if (!coupled) {
    P->vt = VtPath::kNone;
  } else if (nrhs == 1 && p >= 3 && b % 64 == 0 && b <= 4096 && pow2_rank(k, 1, 64)) {
    P->vt = VtPath::kGemv;
    P->tile = 8 * b;
  } else if (nrhs >= 2 && b % 4 == 0 && pow2_rank(k, 16, 64)) {
    P->vt = VtPath::kMma;  // batched: warps per leaf
    P->nt_vt = nt_for(nrhs, HM_VTB_NTMAX);
  } else {
    P->vt = VtPath::kGeneric;
    P->mc_vt = vt_mc(b, nrhs);
    P->tile = pick_tile(b, p, P->mc_vt);
  }
  P->mma_levels = coupled && nrhs >= 2 && pow2_rank(k, 16, 64);
  P->gemv_levels = coupled && nrhs <= kTreeGemvMaxM && pow2_rank(k, 16, 64);
  if (P->mma_levels) P->nt_down = nt_for(nrhs, HM_TREE_NTMAX);
  const int ktot = leaf_coupled ? k : 0;
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
  const size_t blk = sizeof(double) * (size_t)k * nrhs;
  const size_t coef = blk * (size_t)((((int64_t)1 << (p + 1)) - 2));
  const size_t tcoef = blk * (size_t)((((int64_t)1 << (q + 1)) - 2));
  size_t off = 0;
  P->off_xh = off; off = align_up(off + coef);
  P->off_yh = off; off = align_up(off + coef);
  P->off_txh = off; off = align_up(off + tcoef);
  P->off_tyh = off; off = align_up(off + tcoef);
  P->off_x = P->off_y = off;
  if (flags & HM_WS_HOSTIO) {
    P->off_x = off; off = align_up(off + sizeof(double) * (size_t)(n * nrhs));
    P->off_y = off; off = align_up(off + sizeof(double) * (size_t)(n * nrhs));
  }
  P->total = std::max<size_t>(off, kAlign);
  return HM_OK;
}

hm_status hss_plan(const hm_tree* tree, int32_t k, int32_t nrhs, int32_t flags, HssPlan* P) {
  hm_status st = check_tree(tree);
  if (st) return st;
  return hss_plan_ex(tree->n, tree->leaf, tree->levels, 0, k, nrhs, flags, P);
}

// Levels with at least kTreeBigLevel nodes run one launch per level; the
// levels above run inside one cooperative launch (hss_tree_sweep_kernel).
#ifndef HM_TREE_BIG_LEVEL
#define HM_TREE_BIG_LEVEL 2048
#endif
constexpr int64_t kTreeBigLevel = HM_TREE_BIG_LEVEL;

// ---- nrhs <= 4: warp-per-node GEMV tree levels (hm_treegemv.cuh) ----
#ifndef HM_GEMV_BIG
#define HM_GEMV_BIG 8192
#endif
constexpr int64_t kGemvBigLevel = HM_GEMV_BIG;  // nodes: one launch per level from here down

template <int K, int MB>
hm_status tree_gemv_launch(const hm::TreeGemvParams& tp, int p, bool up, bool down, cudaStream_t s, int up_from_l,
                           int down_last) {
  static int64_t cap = -1;  // co-resident CTAs of the sweep kernel (queried once)
  if (cap < 0) {
    int per_sm = 0, dev = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hm::hss_tree_gemv_sweep_kernel<K, MB>, 256, 0) !=
        cudaSuccess)
      return cuda_check("occupancy query (hss_tree_gemv_sweep)");
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cap = (int64_t)per_sm * sms;
  }
  int lbig = 1;  // first level with >= kGemvBigLevel nodes
  while (lbig <= p && (1ll << lbig) < kGemvBigLevel) ++lbig;
  hm_status st;
  for (int l = up_from_l; up && l >= lbig; --l) {
    const unsigned grid = (unsigned)(((1ll << l) + 7) / 8);
    st = launch("hss_up_gemv", s, [&] { hm::hss_up_gemv_kernel<K, MB><<<grid, 256, 0, s>>>(tp, l); });
    if (st) return st;
  }
  const int up_from = up ? std::min(up_from_l, lbig - 1) : 0, down_to = down ? std::min(down_last, lbig - 1) : 0;
  if (up_from >= 1 || down_to >= 1) {
    const int64_t need = std::max<int64_t>(1, ((1ll << std::max(up_from, down_to)) + 7) / 8);
    dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(cap, need)));
    hm::TreeGemvParams arg = tp;
    int a1 = up_from, a2 = down_to;
    void* args[] = {&arg, &a1, &a2};
    cudaError_t e = cudaSuccess;
    st = launch("hss_tree_gemv_sweep", s, [&] {
      e = cudaLaunchCooperativeKernel((const void*)hm::hss_tree_gemv_sweep_kernel<K, MB>, grid, dim3(256), args, 0,
                                      s);
    });
    if (st == HM_OK && e != cudaSuccess) return fail(HM_ERR_CUDA, "hss_tree_gemv_sweep: %s", cudaGetErrorString(e));
    if (st) return st;
  }
  for (int l = std::max(lbig, 1); down && l <= down_last; ++l) {
    const unsigned grid = (unsigned)(((1ll << l) + 7) / 8);
    st = launch("hss_down_gemv", s, [&] { hm::hss_down_gemv_kernel<K, MB><<<grid, 256, 0, s>>>(tp, l); });
    if (st) return st;
  }
  return HM_OK;
}

hm_status tree_gemv_dispatch(const hm::TreeGemvParams& tp, int p, int k, bool up, bool down, cudaStream_t s,
                             int up_from, int down_last) {
  const int mb = tp.m <= 1 ? 1 : (tp.m <= 2 ? 2 : 4);
#define HM_TG(K_)                                                                      \
  if (k == K_) {                                                                       \
    if (mb == 1) return tree_gemv_launch<K_, 1>(tp, p, up, down, s, up_from, down_last); \
    if (mb == 2) return tree_gemv_launch<K_, 2>(tp, p, up, down, s, up_from, down_last); \
    return tree_gemv_launch<K_, 4>(tp, p, up, down, s, up_from, down_last);            \
  }
  HM_TG(16)
  HM_TG(32)
  HM_TG(64)
#undef HM_TG
  return fail(HM_ERR_UNSUPPORTED, "hss tree gemv: no instance for k=%d", k);
}

template <int KT, int NT>
hm_status tree_launch(const hm::TreeParams& tp, int p, bool up, bool down, cudaStream_t s, int up_from_l,
                      int down_last) {
#ifndef HM_TREE_UP_MINB
#define HM_TREE_UP_MINB 4
#endif
#ifndef HM_TREE_DN_MINB
#define HM_TREE_DN_MINB 3
#endif
  // min CTAs per SM for the config-4 shape (k = 32, m = 32), measured (r01_tuning.md)
  constexpr int MINB_UP = (KT == 32 && NT == 4) ? HM_TREE_UP_MINB : 0;
  constexpr int MINB = (KT == 32 && NT == 4) ? HM_TREE_DN_MINB : 0;
  const size_t smem = sizeof(double) * (size_t)hm::tree_smem_doubles(KT, tp.m, NT);
  static bool attrs = false;
  int sweep_blocks_per_sm = 0;
  if (!attrs) {
    allow_smem(hm::hss_up_pair_kernel<KT, NT, MINB_UP>, 200 * 1024);
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
  // upsweep: big levels up_from_l .. lbig one launch each
  for (int l = up_from_l; up && l >= lbig; --l) {
    const unsigned pairs = (unsigned)(1ll << (l - 1));
    st = launch("hss_up_pair", s, [&] { hm::hss_up_pair_kernel<KT, NT, MINB_UP><<<pairs, 256, smem, s>>>(tp, l); });
    if (st) return st;
  }
  // small levels: up min(p-1, lbig-1) .. 1, down 1 .. min(p, lbig-1)
  const int up_from = up ? std::min(up_from_l, lbig - 1) : 0, down_to = down ? std::min(down_last, lbig - 1) : 0;
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
  for (int l = std::max(lbig, 1); down && l <= down_last; ++l) {
    const unsigned pairs = (unsigned)(1ll << (l - 1));
    st = launch("hss_down_pair", s, [&] { hm::hss_down_pair_kernel<KT, NT, MINB><<<pairs, 256, smem, s>>>(tp, l); });
    if (st) return st;
  }
  return HM_OK;
}

hm_status tree_dispatch(const hm::TreeParams& tp, int p, int k, int nt, bool up, bool down, cudaStream_t s,
                        int up_from, int down_last) {
#define HM_TREE(KT_)                                                                     \
  if (k == KT_) {                                                                        \
    if (nt == 1) return tree_launch<KT_, 1>(tp, p, up, down, s, up_from, down_last);     \
    if (nt == 2) return tree_launch<KT_, 2>(tp, p, up, down, s, up_from, down_last);     \
    return tree_launch<KT_, 4>(tp, p, up, down, s, up_from, down_last);                  \
  }
  HM_TREE(16)
  HM_TREE(32)
  HM_TREE(64)
#undef HM_TREE
  return fail(HM_ERR_UNSUPPORTED, "hss tree: no instance for k=%d", k);
}

// Upsweep and coupling/downsweep of a (sub)tree of depth p on its workspace:
// generic per-level kernels or the DMMA tree kernels (tree_dispatch).
hm_status hss_tree_phase(const HssPlan& P, int p, const double* W, const double* R, const double* B, double* xh,
                         double* yh, const double* R_root, const double* y_root, bool up, bool down,
                         cudaStream_t stream, int bt = 0, int up_from = -1, int down_last = -1) {
  const int k = P.k, nrhs = P.m;
  hm_status st;
  if (up_from < 0) up_from = p - 1;  // first upsweep level to compute
  if (down_last < 0) down_last = p;  // last downsweep level to compute
  if (P.gemv_levels) {
    hm::TreeGemvParams tp{W, R, B, xh, yh, R_root, y_root, nrhs, bt};
    return tree_gemv_dispatch(tp, p, k, up, down, stream, up_from, down_last);
  }
  if (P.mma_levels) {
    hm::TreeParams tp{W, R, B, xh, yh, R_root, y_root, nrhs, bt};
    return tree_dispatch(tp, p, k, P.nt_down, up, down, stream, up_from, down_last);
  }
  const int64_t km = (int64_t)k * nrhs;
  if (up)
    for (int l = up_from; l >= 1; --l) {
      hm::HssLevelParams hp{W, B, xh, yh, nullptr, nullptr, l, k, nrhs, 0};
      const int64_t total = ((int64_t)1 << l) * km;
      const unsigned blocks = (unsigned)std::min<int64_t>((total + hm::kThreads - 1) / hm::kThreads, 148 * 16);
      st = launch("hss_up_level", stream, [&] { hm::hss_up_level_kernel<<<blocks, hm::kThreads, 0, stream>>>(hp); });
      if (st) return st;
    }
  if (down)
    for (int l = 1; l <= down_last; ++l) {
      hm::HssLevelParams hp{R, B, xh, yh, R_root, y_root, l, k, nrhs, bt};
      const int64_t total = ((int64_t)1 << l) * km;
      const unsigned blocks = (unsigned)std::min<int64_t>((total + hm::kThreads - 1) / hm::kThreads, 148 * 16);
      st = launch("hss_down_level", stream,
                  [&] { hm::hss_down_level_kernel<<<blocks, hm::kThreads, 0, stream>>>(hp); });
      if (st) return st;
    }
  return HM_OK;
}

// x_out = A^T Z for one block (A [K][k], Z [K][m]): the subtree root's upsweep
// step x_root = W_root^T [x_{1,0}; x_{1,1}] and the leaf-only subtree x = V^T X.
hm_status hss_single_vt(const HssPlan& P, const double* A, const double* Z, int64_t K, double* out,
                        cudaStream_t stream) {
  const int k = P.k, nrhs = P.m;
  if (nrhs >= 2 && pow2_rank(k, 16, 64) && K % 4 == 0) {
    hm::BatchedVtParams bp{A, 0, Z, 0, out, 0, 1, (int32_t)K, nrhs};
    return vt_batched_dispatch("vt_batched", bp, k, nt_for(nrhs, HM_VTB_NTMAX), stream);
  }
  hm::VtParams vp;
  memset(&vp, 0, sizeof vp);
  vp.X = Z; vp.n = K; vp.m = nrhs; vp.mc = vt_mc(K, nrhs); vp.tile = K; vp.nlev = 1;
  vp.lev[0].V = A; vp.lev[0].k = k; vp.lev[0].s = K; vp.lev[0].out = out; vp.lev[0].partial = nullptr;
  return vt_generic(vp, K, stream);
}

// Fused Step 1 + first upsweep level (hss_leaf_up_kernel): k in {16, 32, 64},
// 2 <= m <= 32, leaf a multiple of 16 and two leaves' staging in shared memory.
int leafup_mp(int m) { return m <= 8 ? 8 : (m <= 16 ? 16 : 32); }

template <int KT, int MP>
size_t leafup_smem(int ru, int wd) { return hm::LeafUpLayout<KT, MP>::smem_bytes(ru, wd); }

int leafup_wd(int64_t b, int ru) { return b / ru >= 2 ? 2 : 3; }

size_t leafup_smem_rt(int k, int mp, int ru, int64_t b) {
#define HM_LU(KT_, MP_) if (k == KT_ && mp == MP_) return leafup_smem<KT_, MP_>(ru, leafup_wd(b, ru));
  HM_LU(16, 8) HM_LU(16, 16) HM_LU(16, 32) HM_LU(32, 8) HM_LU(32, 16) HM_LU(32, 32) HM_LU(64, 8) HM_LU(64, 16)
  HM_LU(64, 32)
#undef HM_LU
  return (size_t)-1;
}

// The fused Step-1 + first-upsweep kernel (hm_leafup.cuh) is correct (parity
// tested with HM_LEAFUP=1) but measured slower than vt_batched + hss_up_pair on
// config 4 (763 vs 629 us: a persistent 1-CTA/SM pipeline leaves the DMMA pipe
// 60% idle; r01_tuning.md), so it is off by default.
#ifndef HM_LEAFUP
#define HM_LEAFUP 0
#endif
#define HM_NO_LEAFUP (!HM_LEAFUP)

// Rows per pipeline unit: the largest power of two <= 64 dividing the leaf
// whose 4-slot ring fits in 226 KB of shared memory (0: none fits).
int leafup_ru(const HssPlan& P) {
  for (int ru = 64; ru >= 32; ru >>= 1)  // two contraction halves of >= 16 rows
    if (P.b % ru == 0 && leafup_smem_rt(P.k, leafup_mp(P.m), ru, P.b) <= 226 * 1024) return ru;
  return 0;
}

bool leafup_ok(const HssPlan& P) {
  if (HM_NO_LEAFUP || P.m < 2 || P.m > 32 || P.b % 32 != 0) return false;
  if (!(P.k == 16 || P.k == 32 || P.k == 64)) return false;
  return leafup_ru(P) > 0;
}

template <int KT, int MP>
hm_status leafup_launch(const hm::LeafUpParams& lp, cudaStream_t s) {
  const size_t smem = leafup_smem<KT, MP>(lp.ru, lp.wd);
  allow_smem(hm::hss_leaf_up_kernel<KT, MP>, smem);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(lp.npairs, sms));
  return launch("hss_leaf_up", s,
                [&] { hm::hss_leaf_up_kernel<KT, MP><<<grid, hm::kLeafUpThreads, smem, s>>>(lp); });
}

hm_status leafup_dispatch(const HssPlan& P, const double* V, const double* W, const double* Xd, double* xh,
                          cudaStream_t s) {
  const int ru = leafup_ru(P);
  hm::LeafUpParams lp{V, Xd, P.p >= 2 ? W : nullptr, xh, (int64_t)1 << (P.p - 1), (int32_t)P.b, P.m, P.p,
                      ru, leafup_wd(P.b, ru), 0};
  const int mp = leafup_mp(P.m);
#define HM_LU(KT_, MP_) if (P.k == KT_ && mp == MP_) return leafup_launch<KT_, MP_>(lp, s);
  HM_LU(16, 8) HM_LU(16, 16) HM_LU(16, 32) HM_LU(32, 8) HM_LU(32, 16) HM_LU(32, 32) HM_LU(64, 8) HM_LU(64, 16)
  HM_LU(64, 32)
#undef HM_LU
  return fail(HM_ERR_UNSUPPORTED, "hss_leaf_up: no instance for k=%d m=%d", P.k, P.m);
}

// Step 1 on the subtree: leaf x = V^T X, upsweep to level 1, and (W_root given)
// the subtree root's x_root = W_root^T [x_{1,0}; x_{1,1}]. A depth-0 subtree is
// one leaf: its x is the root's, written to x_root.
hm_status hss_up_phase(const HssPlan& P, const double* V, const double* W, const double* Xd, double* xh,
                       const double* W_root, double* x_root, cudaStream_t stream) {
  const int k = P.k, nrhs = P.m;
  const int64_t km = (int64_t)k * nrhs;
  hm_status st;
  double* xleaf = (P.p == 0) ? x_root : xh + (((int64_t)1 << P.p) - 2) * km;
  if (xleaf == nullptr) return HM_OK;
  int up_from = P.p - 1;
  if (P.vt == VtPath::kMma && P.p >= 1 && leafup_ok(P)) {
    // Step 1 fused with the first upsweep level (hm_leafup.cuh)
    if ((st = leafup_dispatch(P, V, W, Xd, xh, stream))) return st;
    up_from = P.p - 2;
  } else if (P.vt == VtPath::kMma) {
    hm::BatchedVtParams bp{V, P.b * k, Xd, P.b * nrhs, xleaf, km, (int64_t)1 << P.p, (int32_t)P.b, nrhs};
    if ((st = vt_batched_dispatch("vt_batched", bp, k, P.nt_vt, stream))) return st;
  } else {
    hm::VtParams vp;
    memset(&vp, 0, sizeof vp);
    vp.X = Xd; vp.n = P.n; vp.m = nrhs; vp.mc = P.mc_vt ? P.mc_vt : vt_mc(P.b, nrhs);
    vp.tile = P.tile ? P.tile : pick_tile(P.b, P.p, vp.mc); vp.nlev = 1;
    vp.lev[0].V = V; vp.lev[0].k = k; vp.lev[0].s = P.b;
    vp.lev[0].out = xleaf;
    vp.lev[0].partial = nullptr;
    st = (P.vt == VtPath::kGemv) ? vt_gemv_dispatch(vp, P.b, k, stream) : vt_generic(vp, P.n, stream);
    if (st) return st;
  }
  if (up_from >= 1 && (st = hss_tree_phase(P, P.p, W, nullptr, nullptr, xh, nullptr, nullptr, nullptr, true,
                                             false, stream, 0, up_from)))
    return st;
  if (W_root && P.p >= 1 && (st = hss_single_vt(P, W_root, xh, 2 * k, x_root, stream))) return st;
  return HM_OK;
}

// Step 4: Y(I_i) = U_i y_i + D_i X(I_i); y of the leaves from yh (or y_root for a
// depth-0 subtree).
// fused: {B, R, xh, yh} of the tree when the leaf-level coupling + downsweep runs
// inside the DMMA leaf kernel (leaf_mma DOWN; yleaf is then not read).
struct FusedDown {
  const double *B, *R, *xh, *yh;
};

hm_status hss_leaf_phase(const HssPlan& P, const double* D, const double* U, const double* Xd, double* Yd,
                         const double* yleaf, cudaStream_t stream, bool dtrans = false,
                         const FusedDown* fd = nullptr) {
  hm::LeafParams lp;
  memset(&lp, 0, sizeof lp);
  lp.D = D; lp.X = Xd; lp.Y = Yd; lp.b = P.b; lp.m = P.m; lp.mc = P.mc_leaf; lp.dtrans = dtrans ? 1 : 0;
  if (fd) {
    const int64_t km = (int64_t)P.k * P.m, kk = (int64_t)P.k * P.k;
    lp.dp = P.p;
    lp.dB = fd->B + (((int64_t)1 << (P.p - 1)) - 1) * 2 * kk;                 // level p-1 nodes' cores
    lp.dR = P.p >= 2 ? fd->R + (((int64_t)1 << (P.p - 1)) - 2) * 2 * kk : nullptr;
    lp.dx = fd->xh + (((int64_t)1 << P.p) - 2) * km;                            // level p x blocks
    lp.dyp = P.p >= 2 ? fd->yh + (((int64_t)1 << (P.p - 1)) - 2) * km : nullptr;  // level p-1 y blocks
  }
  const bool coupled = P.k > 0 && yleaf != nullptr;
  if (coupled) {
    hm::LeafSeg& sg = lp.seg[lp.nseg++];
    sg.A = U;
    sg.T = yleaf;
    sg.k = P.k; sg.shift = 0; sg.xr = 0;
    lp.ktot = P.k;
  }
  return leaf_dispatch(lp, 1ll << P.p, P.leaf, coupled ? P.k : 0, P.nt_leaf, P.mc_leaf, stream);
}

hm_status hss_check_ptrs(const HssPlan& P, const double* U, const double* V, const double* R, const double* W,
                         const double* B, void* ws, size_t ws_bytes) {
  if (!ws || ws_bytes < P.total) return fail(HM_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, P.total);
  if (!aligned16(ws)) return fail(HM_ERR_INVALID_ARG, "workspace must be 16-byte aligned");
  const int k = P.k;
  if (k == 0 || P.p + P.q == 0) return HM_OK;  // block diagonal: only D is read
  if (!U || !V) return fail(HM_ERR_INVALID_ARG, "NULL U / V pointer");
  if (P.p > 0 && !B) return fail(HM_ERR_INVALID_ARG, "NULL B pointer");
  if (P.p > 1 && (!R || !W)) return fail(HM_ERR_INVALID_ARG, "NULL R / W pointer");
  if (k > 0 && (!aligned16(U) || !aligned16(V) || (B && !aligned16(B)) || (R && !aligned16(R)) || (W && !aligned16(W))))
    return fail(HM_ERR_INVALID_ARG, "U, V, R, W, B must be 16-byte aligned");
  return HM_OK;
}

// Leaf-level coupling + downsweep fused into the DMMA leaf kernel (leaf_mma
// DOWN): correct (parity tested with HM_FUSED_DOWN=1) but measured slower on
// config 4 — the leaf kernel grows by 457 us (the y_i product sits on each CTA's
// critical path before the main product) while the level-p down kernel saves
// 230 us (r01_tuning.md). Off by default.
#ifndef HM_FUSED_DOWN
#define HM_FUSED_DOWN 0
#endif
#define HM_NO_FUSED_DOWN (!HM_FUSED_DOWN)

// ---- small trees: one cooperative launch (hm_small.cuh) ----
#ifndef HM_NO_SMALL
#define HM_NO_SMALL 0
#endif
constexpr int kSmallMaxLevels = 8;  // up to 256 leaves: one CTA per leaf, all co-resident

bool small_ok(const HssPlan& P) {
  return !HM_NO_SMALL && P.q == 0 && P.mma_levels && P.p >= 1 && P.p <= kSmallMaxLevels && P.m >= 2 && P.m <= 32 &&
         (P.b == 64 || P.b == 128);
}

template <int KT, int NT, int RG>
hm_status small_launch(const hm::SmallHssParams& sp, unsigned grid, cudaStream_t s) {
  const size_t smem = sizeof(double) * (size_t)KT * (NT * 8 + 2);
  static int64_t cap = -1;  // co-resident CTAs of this instance (queried once)
  if (cap < 0) {
    int per_sm = 0, dev = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hm::hss_small_kernel<KT, NT, RG>, 256, smem) !=
        cudaSuccess)
      return cuda_check("occupancy query (hss_small)");
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cap = (int64_t)per_sm * sms;
  }
  if (cap < (int64_t)grid) return fail(HM_ERR_UNSUPPORTED, "hss_small: grid not co-resident");
  hm::SmallHssParams arg = sp;
  void* args[] = {&arg};
  cudaError_t e = cudaSuccess;
  hm_status st = launch("hss_small", s, [&] {
    e = cudaLaunchCooperativeKernel((const void*)hm::hss_small_kernel<KT, NT, RG>, dim3(grid), dim3(256), args, smem,
                                    s);
  });
  if (st == HM_OK && e != cudaSuccess) return fail(HM_ERR_CUDA, "hss_small: %s", cudaGetErrorString(e));
  return st;
}

hm_status small_dispatch(const HssPlan& P, const double* D, const double* U, const double* V, const double* R,
                         const double* W, const double* B, const double* X, double* Y, double* xh, double* yh,
                         cudaStream_t s) {
  const int h = std::min(3, P.p);
  hm::SmallHssParams sp{D, U, V, R, W, B, X, Y, xh, yh, (int32_t)P.b, P.p, P.m, h, 1 << (P.p - h), 0};
  const unsigned grid = 1u << P.p;
  const int nt = P.m <= 16 ? 2 : 4, rg = (int)(P.b / 64);
#define HM_SM(KT_)                                                         \
  if (P.k == KT_) {                                                        \
    if (nt == 2 && rg == 1) return small_launch<KT_, 2, 1>(sp, grid, s);   \
    if (nt == 2 && rg == 2) return small_launch<KT_, 2, 2>(sp, grid, s);   \
    if (nt == 4 && rg == 1) return small_launch<KT_, 4, 1>(sp, grid, s);   \
    if (nt == 4 && rg == 2) return small_launch<KT_, 4, 2>(sp, grid, s);   \
  }
  HM_SM(16)
  HM_SM(32)
  HM_SM(64)
#undef HM_SM
  return fail(HM_ERR_UNSUPPORTED, "hss_small: no instance");
}

// op = 1: Y = A^T X. A^T is HSS on the same tree with row
// bases V (translations W), column bases U (translations R), cores
// S'_{2q,2q+1} = B21^T, S'_{2q+1,2q} = B12^T and leaf blocks D_i^T: the same
// four steps with U <-> V, R <-> W exchanged, transposed cores (bt) and D^T.
hm_status hss_run(const hm_tree* tree, int32_t k, const double* D, const double* U, const double* V,
                  const double* R, const double* W, const double* B, const double* X, int32_t nrhs, double* Y,
                  void* ws, size_t ws_bytes, cudaStream_t stream, int32_t flags, int op = 0) {
  if (op) {
    std::swap(U, V);
    std::swap(R, W);
  }
  HssPlan P;
  hm_status st = hss_plan(tree, k, nrhs, flags, &P);
  if (st) return st;
  if (!D || !X || !Y) return fail(HM_ERR_INVALID_ARG, "NULL D / X / Y pointer");
  if (!aligned16(D)) return fail(HM_ERR_INVALID_ARG, "D must be 16-byte aligned");
  if ((st = hss_check_ptrs(P, U, V, R, W, B, ws, ws_bytes))) return st;
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
  if (coupled && op == 0 && small_ok(P)) {  // small tree: the whole product in one launch (hm_small.cuh)
    if ((st = small_dispatch(P, D, U, V, R, W, B, Xd, Yd, xh, yh, stream)) == HM_OK) {
      if ((flags & HM_WS_HOSTIO) && cudaMemcpyAsync(Y, Yd, xy_bytes, cudaMemcpyDeviceToHost, stream) != cudaSuccess)
        return cuda_check("D2H copy of Y");
      return HM_OK;
    }
    if (st != HM_ERR_UNSUPPORTED) return st;  // not co-resident on this device: the level-by-level path
  }
  // the leaf-level coupling + downsweep fused into the DMMA leaf kernel (forward product)
  const bool fuse = coupled && op == 0 && !HM_NO_FUSED_DOWN && P.leaf == LeafPath::kMma && P.mma_levels;
  if (coupled) {
    if ((st = hss_up_phase(P, V, W, Xd, xh, nullptr, nullptr, stream))) return st;
    if ((!fuse || P.p >= 2) &&
        (st = hss_tree_phase(P, P.p, W, R, B, xh, yh, nullptr, nullptr, false, true, stream, op, -1,
                             fuse ? P.p - 1 : P.p)))
      return st;
  }
  const double* yleaf = coupled ? yh + (((int64_t)1 << P.p) - 2) * km : nullptr;
  const FusedDown fd{B, R, xh, yh};
  if ((st = hss_leaf_phase(P, D, U, Xd, Yd, yleaf, stream, op != 0, fuse ? &fd : nullptr))) return st;
  if (flags & HM_WS_HOSTIO) {
    if (cudaMemcpyAsync(Y, Yd, xy_bytes, cudaMemcpyDeviceToHost, stream) != cudaSuccess)
      return cuda_check("D2H copy of Y");
  }
  return HM_OK;
}

// ---- distributed HSS ----

hm_status hss_dist_plan(const hm_tree* tree, int32_t k, int32_t nrhs, const hm_part* part, int32_t flags,
                        HssPlan* P, DistPart* d) {
  hm_status st = check_tree(tree);
  if (st) return st;
  if ((st = check_part(tree, part, d))) return st;
  return hss_plan_ex(tree->n >> d->q, tree->leaf, tree->levels - d->q, d->q, k, nrhs, flags, P);
}

// ------------------------------------------- general trees (f4) --
//
// Leaf endpoint vector c (host array of 2^p int64): leaf i holds rows
// [c[i-1], c[i]) (c[-1] = 0), possibly empty; D_i blocks concatenated. The host
// derives the row offsets, D offsets and the chunk tables of the V^T X pass and
// copies them into the workspace (one pageable H2D copy per call: general-tree
// calls are not CUDA-graph capturable). HODLR ranks may differ per level.

struct GenPlan {
  int64_t n;
  int32_t p, m, mc_vt, mc_leaf;
  int32_t kmax, ktot;
  int64_t smax;          // largest leaf
  int64_t nchunks;
  // host tables (copied into the workspace at off_tab)
  std::vector<int64_t> lo, doff;
  std::vector<hm::GenChunk> chunks;
  std::vector<int64_t> cbeg;           // all levels back to back
  std::vector<int64_t> cbeg_off;       // per vt level: offset into cbeg
  std::vector<int64_t> chunk0;         // per vt level: first global chunk
  std::vector<int32_t> vt_levels;      // tree level of each vt level (HODLR: 1..p with k > 0; HSS: p)
  size_t off_tab, off_lo, off_doff, off_chunks, off_cbeg;
  size_t off_t[hm::kMaxLevels + 1];    // HODLR t_l blocks
  size_t off_part[hm::kMaxLevels + 1]; // partials per vt level
  size_t tab_bytes, total;
};

hm_status gen_tree(int64_t n, int32_t p, const int64_t* c, GenPlan* G) {
  if (n < 1 || p < 0 || p > 30) return fail(HM_ERR_INVALID_ARG, "general tree: need n >= 1, 0 <= levels <= 30");
  if (p + 1 > hm::kMaxLevels) return fail(HM_ERR_UNSUPPORTED, "too many levels");
  if (!c) return fail(HM_ERR_INVALID_ARG, "endpoint vector c is NULL");
  const int64_t nl = (int64_t)1 << p;
  G->n = n; G->p = p;
  G->lo.assign(nl + 1, 0);
  G->doff.assign(nl, 0);
  int64_t prev = 0, d = 0, smax = 0;
  for (int64_t i = 0; i < nl; ++i) {
    if (c[i] < prev) return fail(HM_ERR_INVALID_ARG, "endpoint vector not nondecreasing at leaf %lld", (long long)i);
    G->lo[i] = prev;
    G->doff[i] = d;
    const int64_t s = c[i] - prev;
    d += s * s;
    smax = std::max(smax, s);
    prev = c[i];
  }
  if (prev != n) return fail(HM_ERR_INVALID_ARG, "last endpoint %lld != n = %lld", (long long)prev, (long long)n);
  G->lo[nl] = n;
  G->smax = smax;
  return HM_OK;
}

// Chunk table of one V^T X level: nodes of tree level l, each split into pieces of
// at most kChunkRows rows (at least one piece, so an empty node gets t = 0).
void gen_add_vt_level(GenPlan* G, int l) {
  const int p = G->p;
  const int64_t nodes = (int64_t)1 << l;
  const int32_t L = (int32_t)G->vt_levels.size();
  G->vt_levels.push_back(l);
  G->cbeg_off.push_back((int64_t)G->cbeg.size());
  G->chunk0.push_back((int64_t)G->chunks.size());
  int64_t rel = 0;
  for (int64_t j = 0; j < nodes; ++j) {
    G->cbeg.push_back(rel);
    const int64_t a = G->lo[j << (p - l)], b = G->lo[(j + 1) << (p - l)];
    const int64_t cnt = std::max<int64_t>(1, (b - a + hm::kChunkRows - 1) / hm::kChunkRows);
    for (int64_t q = 0; q < cnt; ++q) {
      hm::GenChunk ch;
      ch.lo = a + q * hm::kChunkRows;
      ch.hi = std::min(b, ch.lo + hm::kChunkRows);
      if (ch.lo > b) ch.lo = b;
      ch.pidx = (int64_t)G->chunks.size();
      ch.lev = L;
      ch.pad = 0;
      G->chunks.push_back(ch);
      ++rel;
    }
  }
  G->cbeg.push_back(rel);
}

int pick_gen_mc(int64_t smax, int64_t ktot, int32_t m) {
  int mc = 1;
  while (mc < hm::kMaxMc && mc < m) mc <<= 1;
  while (mc > 1 && (smax + ktot) * hm::gen_leaf_zs(mc) > kSmemBudgetDoubles) mc >>= 1;
  return mc;
}

// Tables first (8-byte aligned records, 256-byte aligned regions), then the
// caller's blocks: layout of the table region.
void gen_layout_tables(GenPlan* G, size_t* off) {
  G->off_tab = *off;
  size_t o = 0;
  G->off_lo = o; o = align_up(o + sizeof(int64_t) * G->lo.size());
  G->off_doff = o; o = align_up(o + sizeof(int64_t) * G->doff.size());
  G->off_chunks = o; o = align_up(o + sizeof(hm::GenChunk) * G->chunks.size());
  G->off_cbeg = o; o = align_up(o + sizeof(int64_t) * G->cbeg.size());
  G->tab_bytes = o;
  *off = align_up(*off + o);
  G->nchunks = (int64_t)G->chunks.size();
}

hm_status gen_upload_tables(const GenPlan& G, char* w, cudaStream_t s) {
  thread_local std::vector<char> img;
  img.assign(G.tab_bytes, 0);
  memcpy(img.data() + G.off_lo, G.lo.data(), sizeof(int64_t) * G.lo.size());
  memcpy(img.data() + G.off_doff, G.doff.data(), sizeof(int64_t) * G.doff.size());
  memcpy(img.data() + G.off_chunks, G.chunks.data(), sizeof(hm::GenChunk) * G.chunks.size());
  memcpy(img.data() + G.off_cbeg, G.cbeg.data(), sizeof(int64_t) * G.cbeg.size());
  if (cudaMemcpyAsync(w + G.off_tab, img.data(), G.tab_bytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return cuda_check("H2D copy of the tree tables");
  return HM_OK;
}

// V^T X for every vt level: chunk partials then fixed-order per-node sums.
// `Vlev[L]`, `outlev[L]`, `klev[L]` per vt level.
template <int KT, int NT>
hm_status gen_vt_mma_launch(const hm::GenVtParams& vp, int64_t nchunks, cudaStream_t s) {
  const size_t smem = sizeof(double) * (size_t)(8 * KT * NT * 8);
  allow_smem(hm::gen_vt_mma_kernel<KT, NT>, smem);
  dim3 grid((unsigned)nchunks, (unsigned)((vp.m + NT * 8 - 1) / (NT * 8)));
  return launch("gen_vt_mma", s, [&] { hm::gen_vt_mma_kernel<KT, NT><<<grid, hm::kThreads, smem, s>>>(vp); });
}

hm_status gen_vt_mma_dispatch(const hm::GenVtParams& vp, int64_t nchunks, int k, cudaStream_t s) {
  if (k == 16) return vp.m <= 16 ? gen_vt_mma_launch<16, 2>(vp, nchunks, s) : gen_vt_mma_launch<16, 4>(vp, nchunks, s);
  if (k == 32) return vp.m <= 16 ? gen_vt_mma_launch<32, 2>(vp, nchunks, s) : gen_vt_mma_launch<32, 4>(vp, nchunks, s);
  return gen_vt_mma_launch<64, 2>(vp, nchunks, s);
}

hm_status gen_vt_phase(const GenPlan& G, const double* const* Vlev, double* const* outlev, const int32_t* klev,
                       const double* X, char* w, cudaStream_t s) {
  const int nlev = (int)G.vt_levels.size();
  if (nlev == 0) return HM_OK;
  hm::GenVtParams vp;
  memset(&vp, 0, sizeof vp);
  vp.X = X;
  vp.chunks = reinterpret_cast<const hm::GenChunk*>(w + G.off_tab + G.off_chunks);
  vp.nchunks = G.nchunks;
  vp.m = G.m;
  vp.mc = G.mc_vt;
  vp.nlev = nlev;
  hm::GenReduceParams rp;
  memset(&rp, 0, sizeof rp);
  rp.nlev = nlev;
  rp.m = G.m;
  const int64_t* cbeg_dev = reinterpret_cast<const int64_t*>(w + G.off_tab + G.off_cbeg);
  for (int L = 0; L < nlev; ++L) {
    hm::GenVtLevel& lv = vp.lev[L];
    lv.V = Vlev[L];
    lv.out = outlev[L];
    lv.partial = reinterpret_cast<double*>(w + G.off_part[L]);
    lv.cbeg = cbeg_dev + G.cbeg_off[L];
    lv.nodes = (int64_t)1 << G.vt_levels[L];
    lv.chunk0 = G.chunk0[L];
    lv.k = klev[L];
    rp.lev[L] = lv;
    rp.thread_begin[L] = rp.threads;
    rp.threads += lv.nodes * (int64_t)lv.k * G.m;
  }
  rp.thread_begin[nlev] = rp.threads;
  // nrhs = 1 with even power-of-two ranks: 128-bit streaming GEMV per chunk
  bool gemv = G.m == 1;
  for (int L = 0; L < nlev; ++L) gemv = gemv && pow2_rank(klev[L], 2, 64);
  dim3 grid((unsigned)G.nchunks, (unsigned)((G.m + G.mc_vt - 1) / G.mc_vt));
  // nrhs >= 2 with one rank in {16, 32, 64} on every level: DMMA per chunk
  int kmma = G.m >= 2 ? klev[0] : 0;
  for (int L = 0; L < nlev; ++L) kmma = (klev[L] == kmma && pow2_rank(kmma, 16, 64)) ? kmma : 0;
  hm_status st;
  if (gemv) {
    st = launch("gen_vt_gemv", s, [&] { hm::gen_vt_gemv_kernel<<<(unsigned)G.nchunks, hm::kThreads, 0, s>>>(vp); });
  } else if (kmma) {
    st = gen_vt_mma_dispatch(vp, G.nchunks, kmma, s);
  } else {
    st = launch("gen_vt_chunk", s, [&] { hm::gen_vt_chunk_kernel<<<grid, hm::kThreads, 0, s>>>(vp); });
  }
  if (st) return st;
  const unsigned rg = (unsigned)((rp.threads + hm::kThreads - 1) / hm::kThreads);
  return launch("gen_vt_reduce", s, [&] { hm::gen_vt_reduce_kernel<<<rg, hm::kThreads, 0, s>>>(rp); });
}

template <int MC>
hm_status gen_leaf_launch(const hm::GenLeafParams& lp, int64_t nleaves, int64_t smax, cudaStream_t s) {
  const size_t smem = sizeof(double) * (size_t)((smax + lp.ktot) * hm::gen_leaf_zs(MC));
  allow_smem(hm::gen_leaf_kernel<MC>, std::max<size_t>(smem, 1));
  dim3 grid((unsigned)nleaves, (unsigned)((lp.m + MC - 1) / MC));
  return launch(lp.dtrans ? "gen_leaf_t" : "gen_leaf", s,
                [&] { hm::gen_leaf_kernel<MC><<<grid, hm::kThreads, smem, s>>>(lp); });
}

#ifndef HM_GEN_LEAF_MMA_MIN_M
#define HM_GEN_LEAF_MMA_MIN_M 2
#endif
template <int NT, bool DT>
hm_status gen_leaf_mma_launch(const hm::GenLeafParams& lp, int64_t nleaves, int64_t smax, cudaStream_t s) {
  const size_t smem = sizeof(double) * (size_t)((smax + lp.ktot) * (NT * 8 + 4));
  allow_smem(hm::gen_leaf_mma_kernel<NT, DT>, std::max<size_t>(smem, 1));
  dim3 grid((unsigned)nleaves, (unsigned)((lp.m + NT * 8 - 1) / (NT * 8)));
  return launch(DT ? "gen_leaf_mma_t" : "gen_leaf_mma", s,
                [&] { hm::gen_leaf_mma_kernel<NT, DT><<<grid, hm::kThreads, smem, s>>>(lp); });
}

hm_status gen_leaf_phase(const GenPlan& G, const hm::GenLeafParams& lp, cudaStream_t s) {
  const int64_t nl = (int64_t)1 << G.p;
  // nrhs >= 2: DMMA leaf pass (8 NT columns per CTA) when the staged rows fit
  if (G.m >= HM_GEN_LEAF_MMA_MIN_M) {
    const int nt = G.m <= 8 ? 1 : (G.m <= 16 ? 2 : 4);
    if ((G.smax + G.ktot) * (nt * 8 + 4) <= kSmemBudgetDoubles) {
      if (nt == 1) return lp.dtrans ? gen_leaf_mma_launch<1, true>(lp, nl, G.smax, s) : gen_leaf_mma_launch<1, false>(lp, nl, G.smax, s);
      if (nt == 2) return lp.dtrans ? gen_leaf_mma_launch<2, true>(lp, nl, G.smax, s) : gen_leaf_mma_launch<2, false>(lp, nl, G.smax, s);
      return lp.dtrans ? gen_leaf_mma_launch<4, true>(lp, nl, G.smax, s) : gen_leaf_mma_launch<4, false>(lp, nl, G.smax, s);
    }
  }
  switch (G.mc_leaf) {
    case 1: return gen_leaf_launch<1>(lp, nl, G.smax, s);
    case 2: return gen_leaf_launch<2>(lp, nl, G.smax, s);
    case 4: return gen_leaf_launch<4>(lp, nl, G.smax, s);
    case 8: return gen_leaf_launch<8>(lp, nl, G.smax, s);
    default: return gen_leaf_launch<16>(lp, nl, G.smax, s);
  }
}

hm_status hodlr_gen_plan(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks, int32_t nrhs, GenPlan* G) {
  if (nrhs < 1) return fail(HM_ERR_INVALID_ARG, "nrhs = %d < 1", nrhs);
  hm_status st = gen_tree(n, p, c, G);
  if (st) return st;
  if (p > 0 && !ranks) return fail(HM_ERR_INVALID_ARG, "ranks is NULL");
  G->m = nrhs;
  G->kmax = 0; G->ktot = 0;
  for (int l = 1; l <= p; ++l) {
    if (ranks[l - 1] < 0) return fail(HM_ERR_INVALID_ARG, "ranks[%d] = %d < 0", l - 1, ranks[l - 1]);
    if (ranks[l - 1] > hm::kMaxRank) return fail(HM_ERR_UNSUPPORTED, "rank %d > %d", ranks[l - 1], hm::kMaxRank);
    G->kmax = std::max(G->kmax, ranks[l - 1]);
    G->ktot += ranks[l - 1];
    if (ranks[l - 1] > 0) gen_add_vt_level(G, l);
  }
  if ((G->smax + G->ktot) > kSmemBudgetDoubles)
    return fail(HM_ERR_UNSUPPORTED, "largest leaf %lld + ranks %d too large for shared-memory staging",
                (long long)G->smax, G->ktot);
  G->mc_vt = std::max(1, std::min<int>(nrhs, hm::kThreads / std::max(1, G->kmax)));
  G->mc_leaf = pick_gen_mc(G->smax, G->ktot, nrhs);
  size_t off = 0;
  gen_layout_tables(G, &off);
  for (int l = 1; l <= p; ++l) {
    G->off_t[l] = off;
    off = align_up(off + sizeof(double) * (size_t)(((int64_t)1 << l) * ranks[l - 1] * nrhs));
  }
  for (size_t L = 0; L < G->vt_levels.size(); ++L) {
    const int l = G->vt_levels[L];
    G->off_part[L] = off;
    const int64_t cnt = (L + 1 < G->vt_levels.size() ? G->chunk0[L + 1] : G->nchunks) - G->chunk0[L];
    off = align_up(off + sizeof(double) * (size_t)(cnt * ranks[l - 1] * nrhs));
  }
  G->total = std::max<size_t>(off, kAlign);
  return HM_OK;
}

hm_status hodlr_gen_run(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks, int op, const double* D,
                        const double* U, const double* V, const double* X, int32_t nrhs, double* Y, void* ws,
                        size_t ws_bytes, cudaStream_t s) {
  GenPlan G;
  hm_status st = hodlr_gen_plan(n, p, c, ranks, nrhs, &G);
  if (st) return st;
  if (!ws || ws_bytes < G.total) return fail(HM_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, G.total);
  if (!aligned16(ws)) return fail(HM_ERR_INVALID_ARG, "workspace must be 16-byte aligned");
  if (!X || !Y || (!D && G.doff.size() > 0 && n > 0) || (G.ktot > 0 && (!U || !V)))
    return fail(HM_ERR_INVALID_ARG, "NULL generator / X / Y pointer");
  const size_t xy = sizeof(double) * (size_t)(n * nrhs);
  if (overlap(X, xy, Y, xy)) return fail(HM_ERR_INVALID_ARG, "X and Y overlap");
  if (op) std::swap(U, V);  // A^T: HODLR with U and V exchanged, D_i^T
  char* w = static_cast<char*>(ws);
  g_launches = 0;
  prof_new_call();
  if ((st = gen_upload_tables(G, w, s))) return st;
  std::vector<const double*> Vl;
  std::vector<double*> outl;
  std::vector<int32_t> kl;
  int64_t off = 0;
  for (int l = 1; l <= p; ++l) {
    if (ranks[l - 1] > 0) {
      Vl.push_back(V + off);
      outl.push_back(reinterpret_cast<double*>(w + G.off_t[l]));
      kl.push_back(ranks[l - 1]);
    }
    off += n * ranks[l - 1];
  }
  if ((st = gen_vt_phase(G, Vl.data(), outl.data(), kl.data(), X, w, s))) return st;
  hm::GenLeafParams lp;
  memset(&lp, 0, sizeof lp);
  lp.D = D; lp.X = X; lp.Y = Y; lp.m = nrhs; lp.mc = G.mc_leaf; lp.dtrans = op ? 1 : 0;
  lp.lo = reinterpret_cast<const int64_t*>(w + G.off_tab + G.off_lo);
  lp.doff = reinterpret_cast<const int64_t*>(w + G.off_tab + G.off_doff);
  off = 0;
  for (int l = 1; l <= p; ++l) {
    const int k = ranks[l - 1];
    if (k > 0) {
      hm::LeafSeg& sg = lp.seg[lp.nseg++];
      sg.A = U + off;
      sg.T = reinterpret_cast<const double*>(w + G.off_t[l]);
      sg.k = k;
      sg.shift = p - l;
      sg.xr = 1;  // A(I_a, I_sib a) = U_l(I_a) V_l(I_sib a)^T
      lp.ktot += k;
    }
    off += n * k;
  }
  return gen_leaf_phase(G, lp, s);
}

bool ranks_vary(int32_t p, const int32_t* ranks) {
  int k = 0;
  for (int l = 1; l <= p; ++l) {
    if (ranks[l - 1] <= 0) continue;
    if (k != 0 && ranks[l - 1] != k) return true;
    k = ranks[l - 1];
  }
  return false;
}

// Per-level ranks on the uniform tree: the general-tree kernels take
// the call unless every rank fits the tuned kernels (hodlr_plan with kvary).
bool hodlr_use_general(const hm_tree* tree, const int32_t* ranks, int32_t nrhs, int32_t flags) {
  if (!tree || check_tree(tree) != HM_OK || !ranks || !ranks_vary(tree->levels, ranks)) return false;
  HodlrPlan P;
  const std::string saved = g_err;
  const bool fast = hodlr_plan(tree, ranks, nrhs, flags, &P) == HM_OK;
  g_err = saved;
  return !fast;
}

std::vector<int64_t> uniform_endpoints(const hm_tree* t) {
  std::vector<int64_t> c((size_t)1 << t->levels);
  for (size_t i = 0; i < c.size(); ++i) c[i] = (int64_t)(i + 1) * t->leaf;
  return c;
}

// ---- HSS on a general tree ----

hm_status hss_gen_plan(int64_t n, int32_t p, const int64_t* c, int32_t k, int32_t nrhs, GenPlan* G, HssPlan* H) {
  if (nrhs < 1) return fail(HM_ERR_INVALID_ARG, "nrhs = %d < 1", nrhs);
  hm_status st = gen_tree(n, p, c, G);
  if (st) return st;
  // the tree sweeps only see k x m blocks per node: plan them as a uniform tree
  if ((st = hss_plan_ex(((int64_t)1 << p) * 64, 64, p, 0, k, nrhs, 0, H))) return st;
  G->m = nrhs;
  const bool coupled = k > 0 && p > 0;
  G->kmax = k; G->ktot = coupled ? k : 0;
  if (coupled) gen_add_vt_level(G, p);
  if ((G->smax + G->ktot) > kSmemBudgetDoubles)
    return fail(HM_ERR_UNSUPPORTED, "largest leaf %lld too large for shared-memory staging", (long long)G->smax);
  G->mc_vt = std::max(1, std::min<int>(nrhs, hm::kThreads / std::max(1, k)));
  G->mc_leaf = pick_gen_mc(G->smax, G->ktot, nrhs);
  size_t off = 0;
  gen_layout_tables(G, &off);
  const size_t coef = sizeof(double) * (size_t)k * nrhs * (size_t)((((int64_t)1 << (p + 1)) - 2));
  H->off_xh = off; off = align_up(off + coef);
  H->off_yh = off; off = align_up(off + coef);
  if (coupled) {
    G->off_part[0] = off;
    off = align_up(off + sizeof(double) * (size_t)(G->nchunks * k * nrhs));
  }
  G->total = std::max<size_t>(off, kAlign);
  return HM_OK;
}

hm_status hss_gen_run(int64_t n, int32_t p, const int64_t* c, int32_t k, int op, const double* D, const double* U,
                      const double* V, const double* R, const double* W, const double* B, const double* X,
                      int32_t nrhs, double* Y, void* ws, size_t ws_bytes, cudaStream_t s) {
  GenPlan G;
  HssPlan H;
  hm_status st = hss_gen_plan(n, p, c, k, nrhs, &G, &H);
  if (st) return st;
  if (!ws || ws_bytes < G.total) return fail(HM_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, G.total);
  if (!aligned16(ws)) return fail(HM_ERR_INVALID_ARG, "workspace must be 16-byte aligned");
  const bool coupled = k > 0 && p > 0;
  if (!X || !Y || !D) return fail(HM_ERR_INVALID_ARG, "NULL D / X / Y pointer");
  if (coupled && (!U || !V || !B || (p >= 2 && (!R || !W)))) return fail(HM_ERR_INVALID_ARG, "NULL generator pointer");
  const size_t xy = sizeof(double) * (size_t)(n * nrhs);
  if (overlap(X, xy, Y, xy)) return fail(HM_ERR_INVALID_ARG, "X and Y overlap");
  if (op) {  // A^T: U <-> V, R <-> W, transposed cores, D_i^T
    std::swap(U, V);
    std::swap(R, W);
  }
  char* w = static_cast<char*>(ws);
  double* xh = reinterpret_cast<double*>(w + H.off_xh);
  double* yh = reinterpret_cast<double*>(w + H.off_yh);
  const int64_t km = (int64_t)k * nrhs;
  g_launches = 0;
  prof_new_call();
  if ((st = gen_upload_tables(G, w, s))) return st;
  const double* yleaf = nullptr;
  if (coupled) {
    double* xleaf = xh + (((int64_t)1 << p) - 2) * km;
    const double* Vl[1] = {V};
    double* outl[1] = {xleaf};
    const int32_t kl[1] = {k};
    if ((st = gen_vt_phase(G, Vl, outl, kl, X, w, s))) return st;  // Step 1: leaf V^T X
    if (p >= 2 && (st = hss_tree_phase(H, p, W, nullptr, nullptr, xh, nullptr, nullptr, nullptr, true, false, s)))
      return st;  // upsweep
    if ((st = hss_tree_phase(H, p, W, R, B, xh, yh, nullptr, nullptr, false, true, s, op))) return st;
    yleaf = yh + (((int64_t)1 << p) - 2) * km;
  }
  hm::GenLeafParams lp;
  memset(&lp, 0, sizeof lp);
  lp.D = D; lp.X = X; lp.Y = Y; lp.m = nrhs; lp.mc = G.mc_leaf; lp.dtrans = op ? 1 : 0;
  lp.lo = reinterpret_cast<const int64_t*>(w + G.off_tab + G.off_lo);
  lp.doff = reinterpret_cast<const int64_t*>(w + G.off_tab + G.off_doff);
  if (coupled) {
    hm::LeafSeg& sg = lp.seg[lp.nseg++];
    sg.A = U; sg.T = yleaf; sg.k = k; sg.shift = 0; sg.xr = 0;
    lp.ktot = k;
  }
  return gen_leaf_phase(G, lp, s);
}

// ------------------------------------------------ norm estimate (f2) --
//
// Power method on A A^* (SURVEY §8(f) f2), nrhs = 1:
//   v = x0/||x0||; iters times: w = A^T v, eta = ||w|| (-> est), z = A w, v = z/||z||.
// Workspace: [matvec workspace][v: n][w: n][norm partials]; every product is
// libhm's own matvec / adjoint on the same workspace.
struct NormPlan {
  size_t off_v, off_w, off_part, total;
};

NormPlan norm_plan(size_t mv_bytes, int64_t n) {
  NormPlan N;
  size_t off = align_up(mv_bytes);
  N.off_v = off; off = align_up(off + sizeof(double) * (size_t)n);
  N.off_w = off; off = align_up(off + sizeof(double) * (size_t)n);
  N.off_part = off; off = align_up(off + sizeof(double) * hm::kVecMaxBlocks);
  N.total = off;
  return N;
}

template <typename Apply>
hm_status power_norm2(int64_t n, const double* x0, int32_t iters, double* est, char* w, const NormPlan& N,
                      cudaStream_t s, Apply&& apply) {
  if (iters < 1) return fail(HM_ERR_INVALID_ARG, "iters = %d < 1", iters);
  if (!x0 || !est) return fail(HM_ERR_INVALID_ARG, "NULL x0 / est pointer");
  double* v = reinterpret_cast<double*>(w + N.off_v);
  double* wv = reinterpret_cast<double*>(w + N.off_w);
  double* part = reinterpret_cast<double*>(w + N.off_part);
  const int G = hm::vec_blocks(n);
  const unsigned gs = (unsigned)std::min<int64_t>((n + hm::kVecThreads - 1) / hm::kVecThreads, 148 * 8);
  int32_t launches = 0;
  hm_status st;
  auto sumsq = [&](const double* x) {
    ++launches;
    return launch("vec_sumsq", s, [&] { hm::vec_sumsq_kernel<<<G, hm::kVecThreads, 0, s>>>(x, n, part); });
  };
  auto normalize = [&](const double* x, double* out) {
    ++launches;
    return launch("vec_normalize", s,
                  [&] { hm::vec_normalize_kernel<<<gs, hm::kVecThreads, 0, s>>>(x, n, part, G, out); });
  };
  if ((st = sumsq(x0)) || (st = normalize(x0, v))) return st;
  for (int32_t j = 1; j <= iters; ++j) {
    if ((st = apply(1, v, wv))) return st;  // w = A^T v
    launches += g_launches;
    if ((st = sumsq(wv))) return st;
    ++launches;
    if ((st = launch("vec_norm_write", s, [&] { hm::vec_norm_write_kernel<<<1, 32, 0, s>>>(part, G, est); })))
      return st;                             // eta = ||w||
    if ((st = apply(0, wv, v))) return st;  // z = A w (into v)
    launches += g_launches;
    if ((st = sumsq(v)) || (st = normalize(v, v))) return st;
  }
  g_launches = launches;
  return HM_OK;
}

}  // namespace

extern "C" {

hm_status hm_hodlr_norm2_workspace_bytes(const hm_tree* tree, const int32_t* ranks, size_t* bytes) {
  if (!bytes) return fail(HM_ERR_INVALID_ARG, "bytes is NULL");
  HodlrPlan P;
  hm_status st = hodlr_plan(tree, ranks, 1, 0, &P);
  if (st) return st;
  *bytes = norm_plan(P.total, P.n).total;
  return HM_OK;
}

hm_status hodlr_norm2_est(const hm_tree* tree, const int32_t* ranks, const double* D, const double* U,
                          const double* V, const double* x0, int32_t iters, double* est, void* workspace,
                          size_t workspace_bytes, void* stream) {
  HodlrPlan P;
  hm_status st = hodlr_plan(tree, ranks, 1, 0, &P);
  if (st) return st;
  const NormPlan N = norm_plan(P.total, P.n);
  if (!workspace || workspace_bytes < N.total)
    return fail(HM_ERR_WORKSPACE, "workspace %zu bytes < required %zu", workspace_bytes, N.total);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return power_norm2(P.n, x0, iters, est, static_cast<char*>(workspace), N, s,
                     [&](int op, const double* x, double* y) {
                       return hodlr_run(tree, ranks, D, U, V, x, 1, y, workspace, P.total, s, 0, op);
                     });
}

hm_status hm_hss_norm2_workspace_bytes(const hm_tree* tree, int32_t k, size_t* bytes) {
  if (!bytes) return fail(HM_ERR_INVALID_ARG, "bytes is NULL");
  HssPlan P;
  hm_status st = hss_plan(tree, k, 1, 0, &P);
  if (st) return st;
  *bytes = norm_plan(P.total, P.n).total;
  return HM_OK;
}

hm_status hss_norm2_est(const hm_tree* tree, int32_t k, const double* D, const double* U, const double* V,
                        const double* R, const double* W, const double* B, const double* x0, int32_t iters,
                        double* est, void* workspace, size_t workspace_bytes, void* stream) {
  HssPlan P;
  hm_status st = hss_plan(tree, k, 1, 0, &P);
  if (st) return st;
  const NormPlan N = norm_plan(P.total, P.n);
  if (!workspace || workspace_bytes < N.total)
    return fail(HM_ERR_WORKSPACE, "workspace %zu bytes < required %zu", workspace_bytes, N.total);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return power_norm2(P.n, x0, iters, est, static_cast<char*>(workspace), N, s,
                     [&](int op, const double* x, double* y) {
                       return hss_run(tree, k, D, U, V, R, W, B, x, 1, y, workspace, P.total, s, 0, op);
                     });
}

hm_status hm_hodlr_workspace_bytes(const hm_tree* tree, const int32_t* ranks, int32_t nrhs, int32_t flags,
                                   size_t* bytes) {
  if (!bytes) return fail(HM_ERR_INVALID_ARG, "bytes is NULL");
  if (flags == 0 && hodlr_use_general(tree, ranks, nrhs, flags)) {
    // per-level ranks: the general-tree kernels on the uniform endpoints
    GenPlan G;
    const std::vector<int64_t> c = uniform_endpoints(tree);
    hm_status st = hodlr_gen_plan(tree->n, tree->levels, c.data(), ranks, nrhs, &G);
    if (st) return st;
    *bytes = G.total;
    return HM_OK;
  }
  HodlrPlan P;
  hm_status st = hodlr_plan(tree, ranks, nrhs, flags, &P);
  if (st) return st;
  *bytes = P.total;
  return HM_OK;
}

hm_status hodlr_matvec(const hm_tree* tree, const int32_t* ranks, const double* D, const double* U,
                       const double* V, const double* X, int32_t nrhs, double* Y, void* workspace,
                       size_t workspace_bytes, void* stream) {
  if (hodlr_use_general(tree, ranks, nrhs, 0)) {
    const std::vector<int64_t> c = uniform_endpoints(tree);
    return hodlr_gen_run(tree->n, tree->levels, c.data(), ranks, 0, D, U, V, X, nrhs, Y, workspace, workspace_bytes,
                         static_cast<cudaStream_t>(stream));
  }
  return hodlr_run(tree, ranks, D, U, V, X, nrhs, Y, workspace, workspace_bytes,
                   static_cast<cudaStream_t>(stream), 0);
}

hm_status hodlr_matvec_hostio(const hm_tree* tree, const int32_t* ranks, const double* D, const double* U,
                              const double* V, const double* X_host, int32_t nrhs, double* Y_host,
                              void* workspace, size_t workspace_bytes, void* stream) {
  return hodlr_run(tree, ranks, D, U, V, X_host, nrhs, Y_host, workspace, workspace_bytes,
                   static_cast<cudaStream_t>(stream), HM_WS_HOSTIO);
}

hm_status hodlr_matvec_t(const hm_tree* tree, const int32_t* ranks, const double* D, const double* U,
                         const double* V, const double* X, int32_t nrhs, double* Y, void* workspace,
                         size_t workspace_bytes, void* stream) {
  if (hodlr_use_general(tree, ranks, nrhs, 0)) {
    const std::vector<int64_t> c = uniform_endpoints(tree);
    return hodlr_gen_run(tree->n, tree->levels, c.data(), ranks, 1, D, U, V, X, nrhs, Y, workspace, workspace_bytes,
                         static_cast<cudaStream_t>(stream));
  }
  return hodlr_run(tree, ranks, D, U, V, X, nrhs, Y, workspace, workspace_bytes,
                   static_cast<cudaStream_t>(stream), 0, 1);
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

hm_status hss_matvec_t(const hm_tree* tree, int32_t k, const double* D, const double* U, const double* V,
                       const double* R, const double* W, const double* B, const double* X, int32_t nrhs,
                       double* Y, void* workspace, size_t workspace_bytes, void* stream) {
  return hss_run(tree, k, D, U, V, R, W, B, X, nrhs, Y, workspace, workspace_bytes,
                 static_cast<cudaStream_t>(stream), 0, 1);
}

hm_status hss_matvec_hostio(const hm_tree* tree, int32_t k, const double* D, const double* U, const double* V,
                            const double* R, const double* W, const double* B, const double* X_host,
                            int32_t nrhs, double* Y_host, void* workspace, size_t workspace_bytes, void* stream) {
  return hss_run(tree, k, D, U, V, R, W, B, X_host, nrhs, Y_host, workspace, workspace_bytes,
                 static_cast<cudaStream_t>(stream), HM_WS_HOSTIO);
}

// ---------------------------------------------------------------- multi-GPU --

hm_status hm_hodlr_dist_sizes(const hm_tree* tree, const int32_t* ranks, int32_t nrhs, const hm_part* part,
                              size_t* ws_bytes, int64_t* send_doubles) {
  HodlrPlan P;
  DistPart d;
  hm_status st = hodlr_dist_plan(tree, ranks, nrhs, part, 0, &P, &d);
  if (st) return st;
  if (ws_bytes) *ws_bytes = P.total;
  if (send_doubles) *send_doubles = P.top_doubles;
  return HM_OK;
}

hm_status hodlr_matvec_dist_begin(const hm_tree* tree, const int32_t* ranks, const hm_part* part,
                                  const double* V_local, const double* X_local, int32_t nrhs, double* send,
                                  void* workspace, size_t workspace_bytes, void* stream) {
  HodlrPlan P;
  DistPart d;
  hm_status st = hodlr_dist_plan(tree, ranks, nrhs, part, 0, &P, &d);
  if (st) return st;
  if (!workspace || workspace_bytes < P.total) return fail(HM_ERR_WORKSPACE, "workspace too small");
  if (!X_local || (P.k > 0 && !V_local) || (P.top_doubles > 0 && !send))
    return fail(HM_ERR_INVALID_ARG, "NULL V / X / send pointer");
  g_launches = 0;
  prof_new_call();
  return hodlr_vt_phase(P, ranks, V_local, X_local, static_cast<char*>(workspace), 1, P.q, send,
                        static_cast<cudaStream_t>(stream));
}

hm_status hodlr_matvec_dist_local(const hm_tree* tree, const int32_t* ranks, const hm_part* part,
                                  const double* V_local, const double* X_local, int32_t nrhs, void* workspace,
                                  size_t workspace_bytes, void* stream) {
  HodlrPlan P;
  DistPart d;
  hm_status st = hodlr_dist_plan(tree, ranks, nrhs, part, 0, &P, &d);
  if (st) return st;
  if (!workspace || workspace_bytes < P.total) return fail(HM_ERR_WORKSPACE, "workspace too small");
  if (!X_local || (P.k > 0 && !V_local)) return fail(HM_ERR_INVALID_ARG, "NULL V / X pointer");
  g_launches = 0;
  prof_new_call();
  return hodlr_vt_phase(P, ranks, V_local, X_local, static_cast<char*>(workspace), P.q + 1, P.q + P.p, nullptr,
                        static_cast<cudaStream_t>(stream));
}

hm_status hodlr_matvec_dist_end(const hm_tree* tree, const int32_t* ranks, const hm_part* part,
                                const double* D_local, const double* U_local, const double* X_local, int32_t nrhs,
                                const double* gathered, double* Y_local, void* workspace, size_t workspace_bytes,
                                void* stream) {
  HodlrPlan P;
  DistPart d;
  hm_status st = hodlr_dist_plan(tree, ranks, nrhs, part, 0, &P, &d);
  if (st) return st;
  if (!D_local || !aligned16(D_local)) return fail(HM_ERR_INVALID_ARG, "D_local NULL or misaligned");
  if ((st = hodlr_check_ptrs(P, D_local, U_local, U_local, X_local, Y_local, workspace, workspace_bytes, 0)))
    return st;
  if (P.top_doubles > 0 && !gathered) return fail(HM_ERR_INVALID_ARG, "NULL gathered pointer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(workspace);
  double* ttop = reinterpret_cast<double*>(w + P.off_ttop);
  g_launches = 0;
  prof_new_call();
  if (P.top_doubles > 0) {
    hm::CombineParams cp;
    memset(&cp, 0, sizeof cp);
    cp.gathered = gathered; cp.out = ttop; cp.per_rank = P.top_doubles; cp.q = d.q; cp.rank = d.rank;
    int64_t off = 0;
    for (int l = 1; l <= d.q; ++l) {
      cp.lev_off[l] = off;
      off += (int64_t)ranks[l - 1] * nrhs;
    }
    cp.lev_off[d.q + 1] = off;
    const unsigned grid = (unsigned)((P.top_doubles + hm::kThreads - 1) / hm::kThreads);
    st = launch("dist_combine", s, [&] { hm::dist_combine_kernel<<<grid, hm::kThreads, 0, s>>>(cp); });
    if (st) return st;
  }
  return hodlr_leaf_phase(P, ranks, D_local, U_local, X_local, Y_local, w, ttop, s);
}

hm_status hm_hss_dist_sizes(const hm_tree* tree, int32_t k, int32_t nrhs, const hm_part* part, size_t* ws_bytes,
                            int64_t* send_doubles) {
  HssPlan P;
  DistPart d;
  hm_status st = hss_dist_plan(tree, k, nrhs, part, 0, &P, &d);
  if (st) return st;
  if (ws_bytes) *ws_bytes = P.total;
  if (send_doubles) *send_doubles = (d.q > 0) ? (int64_t)k * nrhs : 0;
  return HM_OK;
}

hm_status hss_matvec_dist_begin(const hm_tree* tree, int32_t k, const hm_part* part, const double* V_local,
                                const double* W_sub, const double* W_root, const double* X_local, int32_t nrhs,
                                double* send, void* workspace, size_t workspace_bytes, void* stream) {
  HssPlan P;
  DistPart d;
  hm_status st = hss_dist_plan(tree, k, nrhs, part, 0, &P, &d);
  if (st) return st;
  if (!workspace || workspace_bytes < P.total || !aligned16(workspace))
    return fail(HM_ERR_WORKSPACE, "workspace too small or misaligned");
  g_launches = 0;
  prof_new_call();
  if (k == 0) return HM_OK;  // block diagonal: nothing to exchange, no tree
  double* xh = reinterpret_cast<double*>(static_cast<char*>(workspace) + P.off_xh);
  if (d.q == 0) {
    // one rank: the whole tree is local and the exchange is empty; Step 1 and
    // the upsweep to level 1 run here (as in hss_matvec), _end does the rest
    if (P.p == 0) return HM_OK;
    if (!X_local || !V_local || (P.p >= 2 && !W_sub)) return fail(HM_ERR_INVALID_ARG, "NULL V / W / X pointer");
    return hss_up_phase(P, V_local, W_sub, X_local, xh, nullptr, nullptr, static_cast<cudaStream_t>(stream));
  }
  if (!X_local || !V_local || !send || (P.p >= 2 && !W_sub) || (P.p >= 1 && !W_root))
    return fail(HM_ERR_INVALID_ARG, "NULL V / W / X / send pointer");
  return hss_up_phase(P, V_local, W_sub, X_local, xh, W_root, send, static_cast<cudaStream_t>(stream));
}

hm_status hss_matvec_dist_end(const hm_tree* tree, int32_t k, const hm_part* part, const double* D_local,
                              const double* U_local, const double* R_sub, const double* B_sub,
                              const double* R_root, const double* W_top, const double* R_top, const double* B_top,
                              const double* X_local, int32_t nrhs, const double* gathered, double* Y_local,
                              void* workspace, size_t workspace_bytes, void* stream) {
  HssPlan P;
  DistPart d;
  hm_status st = hss_dist_plan(tree, k, nrhs, part, 0, &P, &d);
  if (st) return st;
  if (!D_local || !X_local || !Y_local || !aligned16(D_local))
    return fail(HM_ERR_INVALID_ARG, "NULL or misaligned D / X / Y pointer");
  if (!workspace || workspace_bytes < P.total || !aligned16(workspace))
    return fail(HM_ERR_WORKSPACE, "workspace too small or misaligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(workspace);
  double* xh = reinterpret_cast<double*>(w + P.off_xh);
  double* yh = reinterpret_cast<double*>(w + P.off_yh);
  double* txh = reinterpret_cast<double*>(w + P.off_txh);
  double* tyh = reinterpret_cast<double*>(w + P.off_tyh);
  const int64_t km = (int64_t)k * nrhs;
  g_launches = 0;
  prof_new_call();
  const double* yleaf = nullptr;
  if (k > 0 && d.q == 0 && P.p >= 1) {
    // one rank: coupling + downsweep of the whole (local) tree on the x blocks
    // _begin left in the workspace, then the leaves (as in hss_matvec)
    if (!U_local || !B_sub || (P.p >= 2 && !R_sub)) return fail(HM_ERR_INVALID_ARG, "NULL U / R / B pointer");
    if ((st = hss_tree_phase(P, P.p, nullptr, R_sub, B_sub, xh, yh, nullptr, nullptr, false, true, s))) return st;
    yleaf = yh + (((int64_t)1 << P.p) - 2) * km;
  }
  if (k > 0 && d.q > 0) {
    if (!gathered || !U_local || !B_top || (d.q >= 2 && (!W_top || !R_top)) || (P.p >= 1 && (!R_root || !B_sub)) ||
        (P.p >= 2 && !R_sub))
      return fail(HM_ERR_INVALID_ARG, "NULL gathered / generator pointer");
    // replicated top tree: x of level q from the allgather, up q-1..1, down 1..q
    if (cudaMemcpyAsync(txh + (((int64_t)1 << d.q) - 2) * km, gathered, sizeof(double) * (size_t)(d.P * km),
                        cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return cuda_check("copy of the gathered blocks");
    if ((st = hss_tree_phase(P, d.q, W_top, R_top, B_top, txh, tyh, nullptr, nullptr, true, true, s))) return st;
    const double* y_root = tyh + (((int64_t)1 << d.q) - 2 + d.rank) * km;
    if (P.p >= 1) {
      // the subtree's x blocks were left in this workspace by _begin
      if ((st = hss_tree_phase(P, P.p, nullptr, R_sub, B_sub, xh, yh, R_root, y_root, false, true, s))) return st;
      yleaf = yh + (((int64_t)1 << P.p) - 2) * km;
    } else {
      yleaf = y_root;
    }
  }
  return hss_leaf_phase(P, D_local, U_local, X_local, Y_local, yleaf, s);
}

// ------------------------------------------------------ hss2hodlr (f3) --

hm_status hss_to_hodlr(const hm_tree* tree, int32_t k, const double* U, const double* V, const double* R,
                       const double* W, const double* B, double* Uh, double* Vh, void* stream) {
  hm_status st = check_tree(tree);
  if (st) return st;
  if (k < 0) return fail(HM_ERR_INVALID_ARG, "k = %d < 0", k);
  if (k > hm::kMaxRank) return fail(HM_ERR_UNSUPPORTED, "rank %d > %d", k, hm::kMaxRank);
  const int p = tree->levels;
  const int64_t n = tree->n;
  g_launches = 0;
  prof_new_call();
  if (p == 0 || k == 0) return HM_OK;  // no off-diagonal level / all blocks zero: nothing to write
  if (!U || !V || !B || !Uh || !Vh || (p >= 2 && (!R || !W)))
    return fail(HM_ERR_INVALID_ARG, "NULL generator / output pointer");
  const size_t nk = sizeof(double) * (size_t)n * (size_t)k;
  const size_t out = nk * (size_t)p;
  const size_t tr = sizeof(double) * (size_t)((((int64_t)1 << p) - 2) * 2 * k * k);
  const size_t bb = sizeof(double) * (size_t)((((int64_t)1 << p) - 1) * 2 * k * k);
  if (overlap(Uh, out, Vh, out) || overlap(Uh, out, U, nk) || overlap(Uh, out, V, nk) || overlap(Vh, out, U, nk) ||
      overlap(Vh, out, V, nk) || overlap(Uh, out, B, bb) || overlap(Vh, out, B, bb) ||
      (p >= 2 && (overlap(Uh, out, R, tr) || overlap(Uh, out, W, tr) || overlap(Vh, out, R, tr) ||
                  overlap(Vh, out, W, tr))))
    return fail(HM_ERR_INVALID_ARG, "outputs Uh / Vh overlap each other or an input");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (cudaMemcpyAsync(Uh + (size_t)(p - 1) * n * k, U, nk, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(Vh + (size_t)(p - 1) * n * k, V, nk, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return cuda_check("copy of the leaf bases");
  hm::ConvertParams cp{R, W, B, Uh, Vh, n, tree->leaf, p, k};
  if (tree->leaf % 64 == 0 && (k == 16 || k == 32 || k == 64)) {  // one-pass DMMA kernel
    const unsigned g = (unsigned)(n / 64);
    const size_t sm = sizeof(double) * 3 * (size_t)k * (k + 2);
    if (k == 16) return launch("hss2hodlr_mma", s, [&] { hm::hss2hodlr_mma_kernel<16><<<g, 256, sm, s>>>(cp); });
    if (k == 32) return launch("hss2hodlr_mma", s, [&] { hm::hss2hodlr_mma_kernel<32><<<g, 256, sm, s>>>(cp); });
    allow_smem(hm::hss2hodlr_mma_kernel<64>, sm);
    return launch("hss2hodlr_mma", s, [&] { hm::hss2hodlr_mma_kernel<64><<<g, 256, sm, s>>>(cp); });
  }
  const size_t smem = sizeof(double) * 2 * hm::kConvRows * (size_t)k;
  const unsigned grid = (unsigned)((n + hm::kConvRows - 1) / hm::kConvRows);
  for (int l = p; l >= 1; --l) {
    st = launch("hss2hodlr_level", s, [&] { hm::hss2hodlr_level_kernel<<<grid, 256, smem, s>>>(cp, l); });
    if (st) return st;
  }
  return HM_OK;
}

// ---------------------------------------------------- general trees (f4) --

hm_status hm_hodlr_general_workspace_bytes(int64_t n, int32_t levels, const int64_t* c, const int32_t* ranks,
                                           int32_t nrhs, size_t* bytes) {
  if (!bytes) return fail(HM_ERR_INVALID_ARG, "bytes is NULL");
  GenPlan G;
  hm_status st = hodlr_gen_plan(n, levels, c, ranks, nrhs, &G);
  if (st) return st;
  *bytes = G.total;
  return HM_OK;
}

hm_status hodlr_matvec_general(int64_t n, int32_t levels, const int64_t* c, const int32_t* ranks, int32_t op,
                               const double* D, const double* U, const double* V, const double* X, int32_t nrhs,
                               double* Y, void* workspace, size_t workspace_bytes, void* stream) {
  if (op != 0 && op != 1) return fail(HM_ERR_INVALID_ARG, "op = %d (0: A X, 1: A^T X)", op);
  return hodlr_gen_run(n, levels, c, ranks, op, D, U, V, X, nrhs, Y, workspace, workspace_bytes,
                       static_cast<cudaStream_t>(stream));
}

hm_status hm_hss_general_workspace_bytes(int64_t n, int32_t levels, const int64_t* c, int32_t k, int32_t nrhs,
                                         size_t* bytes) {
  if (!bytes) return fail(HM_ERR_INVALID_ARG, "bytes is NULL");
  GenPlan G;
  HssPlan H;
  hm_status st = hss_gen_plan(n, levels, c, k, nrhs, &G, &H);
  if (st) return st;
  *bytes = G.total;
  return HM_OK;
}

hm_status hss_matvec_general(int64_t n, int32_t levels, const int64_t* c, int32_t k, int32_t op, const double* D,
                             const double* U, const double* V, const double* R, const double* W, const double* B,
                             const double* X, int32_t nrhs, double* Y, void* workspace, size_t workspace_bytes,
                             void* stream) {
  if (op != 0 && op != 1) return fail(HM_ERR_INVALID_ARG, "op = %d (0: A X, 1: A^T X)", op);
  return hss_gen_run(n, levels, c, k, op, D, U, V, R, W, B, X, nrhs, Y, workspace, workspace_bytes,
                     static_cast<cudaStream_t>(stream));
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
