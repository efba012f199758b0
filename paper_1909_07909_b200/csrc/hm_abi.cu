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

// ------------------------------------------------------------------ HODLR --

struct HodlrPlan {
  int64_t n, b;
  int32_t p, m, k;       // k = the common nonzero rank (0 if all zero)
  int32_t mc_vt, mc_leaf;
  int64_t tile;
  size_t off_t[hm::kMaxLevels + 1];   // coefficient blocks t_l, per level
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
  int64_t ktot = 0;
  for (int l = 1; l <= P->p; ++l) {
    int k = ranks[l - 1];
    if (k < 0) return fail(HM_ERR_INVALID_ARG, "ranks[%d] = %d < 0", l - 1, k);
    if (k > hm::kMaxRank) return fail(HM_ERR_UNSUPPORTED, "rank %d > %d", k, hm::kMaxRank);
    if (k > 0) {
      if (P->k != 0 && P->k != k)
        return fail(HM_ERR_UNSUPPORTED, "per-level ranks differ (%d vs %d); variable ranks (P:264) not built", P->k, k);
      P->k = k;
    }
    ktot += k;
  }
  P->mc_vt = vt_mc(P->b, nrhs);
  P->mc_leaf = pick_mc(P->b, ktot, nrhs);
  if ((P->b + ktot) * P->mc_leaf > kSmemBudgetDoubles)
    return fail(HM_ERR_UNSUPPORTED, "leaf %lld + ranks %lld too large for shared-memory staging", (long long)P->b, (long long)ktot);
  P->tile = pick_tile(P->b, P->p, P->mc_vt);
  size_t off = 0;
  for (int l = 1; l <= P->p; ++l) {
    int64_t k = ranks[l - 1];
    P->off_t[l] = off;
    off = align_up(off + sizeof(double) * (size_t)((1ll << l) * k * nrhs));
  }
  for (int l = 1; l <= P->p; ++l) {
    int64_t k = ranks[l - 1];
    int64_t s = P->n >> l;
    P->off_part[l] = off;
    if (k > 0 && s > P->tile) off = align_up(off + sizeof(double) * (size_t)((P->n / P->tile) * k * nrhs));
  }
  P->off_x = off;
  P->off_y = off;
  if (flags & HM_WS_HOSTIO) {
    P->off_x = off;
    off = align_up(off + sizeof(double) * (size_t)(P->n * nrhs));
    P->off_y = off;
    off = align_up(off + sizeof(double) * (size_t)(P->n * nrhs));
  }
  P->total = std::max<size_t>(off, kAlign);
  return HM_OK;
}

template <int MC>
hm_status launch_leaf(const hm::LeafParams& lp, int64_t nleaves, int m, size_t smem, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(hm::leaf_apply_kernel<MC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  dim3 grid((unsigned)nleaves, (unsigned)((m + MC - 1) / MC));
  int slot = prof_begin("leaf_apply", s);
  hm::leaf_apply_kernel<MC><<<grid, hm::kThreads, smem, s>>>(lp);
  prof_end(slot, s);
  ++g_launches;
  return cuda_check("leaf_apply_kernel");
}

hm_status leaf_apply(const hm::LeafParams& lp, int64_t nleaves, int mc, cudaStream_t s) {
  size_t smem = sizeof(double) * (size_t)((lp.b + lp.ktot) * mc);
  switch (mc) {
    case 1: return launch_leaf<1>(lp, nleaves, lp.m, smem, s);
    case 2: return launch_leaf<2>(lp, nleaves, lp.m, smem, s);
    case 4: return launch_leaf<4>(lp, nleaves, lp.m, smem, s);
    case 8: return launch_leaf<8>(lp, nleaves, lp.m, smem, s);
    default: return launch_leaf<16>(lp, nleaves, lp.m, smem, s);
  }
}

hm_status vt_contract(const hm::VtParams& vp, int64_t n, size_t smem, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(hm::vt_contract_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  dim3 grid((unsigned)(n / vp.tile), (unsigned)((vp.m + vp.mc - 1) / vp.mc));
  int slot = prof_begin("vt_contract", s);
  hm::vt_contract_kernel<<<grid, hm::kThreads, smem, s>>>(vp);
  prof_end(slot, s);
  ++g_launches;
  return cuda_check("vt_contract_kernel");
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
  if (!aligned16(D) || !aligned16(ws)) return fail(HM_ERR_INVALID_ARG, "D and workspace must be 16-byte aligned");
  const size_t xy_bytes = sizeof(double) * (size_t)(P.n * nrhs);
  if (overlap(X, xy_bytes, Y, xy_bytes)) return fail(HM_ERR_INVALID_ARG, "X and Y overlap");

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

  // (1) all levels' V_l^T X in one pass (vt_contract), partials -> reduce
  if (P.k > 0) {
    hm::VtParams vp;
    memset(&vp, 0, sizeof vp);
    vp.X = Xd; vp.n = P.n; vp.m = nrhs; vp.mc = P.mc_vt; vp.tile = P.tile;
    hm::ReduceParams rp;
    memset(&rp, 0, sizeof rp);
    int64_t uoff = 0;
    for (int l = 1; l <= P.p; ++l) {
      int k = ranks[l - 1];
      int64_t s = P.n >> l;
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
        }
      }
      uoff += P.n * k;
    }
    size_t smem = sizeof(double) * (size_t)(P.tile * P.mc_vt + hm::kThreads);
    if ((st = vt_contract(vp, P.n, smem, stream))) return st;
    if (rp.nlev > 0) {
      dim3 grid(64, rp.nlev);
      int slot = prof_begin("reduce_partials", stream);
      hm::reduce_partials_kernel<<<grid, hm::kThreads, 0, stream>>>(rp);
      prof_end(slot, stream);
      ++g_launches;
      if ((st = cuda_check("reduce_partials_kernel"))) return st;
    }
  }

  // (2) per leaf: Y(I_i) = D_i X(I_i) + sum_l U_l(I_i) t_{l, sib(node_l(i))}
  hm::LeafParams lp;
  memset(&lp, 0, sizeof lp);
  lp.D = D; lp.X = Xd; lp.Y = Yd; lp.b = P.b; lp.m = nrhs; lp.mc = P.mc_leaf;
  {
    int64_t uoff = 0;
    for (int l = 1; l <= P.p; ++l) {
      int k = ranks[l - 1];
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
  if ((st = leaf_apply(lp, 1ll << P.p, P.mc_leaf, stream))) return st;

  if (flags & HM_WS_HOSTIO) {
    if (cudaMemcpyAsync(Y, Yd, xy_bytes, cudaMemcpyDeviceToHost, stream) != cudaSuccess)
      return cuda_check("D2H copy of Y");
  }
  return HM_OK;
}

// -------------------------------------------------------------------- HSS --

struct HssPlan {
  int64_t n, b;
  int32_t p, m, k, mc_vt, mc_leaf;
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
  P->mc_vt = vt_mc(P->b, nrhs);
  P->mc_leaf = pick_mc(P->b, k, nrhs);
  if ((P->b + k) * P->mc_leaf > kSmemBudgetDoubles)
    return fail(HM_ERR_UNSUPPORTED, "leaf %lld too large for shared-memory staging", (long long)P->b);
  P->tile = pick_tile(P->b, P->p, P->mc_vt);
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
  const size_t xy_bytes = sizeof(double) * (size_t)(P.n * nrhs);
  if (overlap(X, xy_bytes, Y, xy_bytes)) return fail(HM_ERR_INVALID_ARG, "X and Y overlap");

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
  const bool coupled = (k > 0 && P.p > 0);
  if (coupled) {
    // Step 1: v_i^p = V_i^T X(I_i) for every leaf (node size b: always complete)
    hm::VtParams vp;
    memset(&vp, 0, sizeof vp);
    vp.X = Xd; vp.n = P.n; vp.m = nrhs; vp.mc = P.mc_vt; vp.tile = P.tile; vp.nlev = 1;
    vp.lev[0].V = V; vp.lev[0].k = k; vp.lev[0].s = P.b;
    vp.lev[0].out = xh + (((int64_t)1 << P.p) - 2) * k * nrhs;
    vp.lev[0].partial = nullptr;
    size_t smem = sizeof(double) * (size_t)(P.tile * P.mc_vt + hm::kThreads);
    if ((st = vt_contract(vp, P.n, smem, stream))) return st;
    // Step 1 (cont.): upsweep l = p-1 .. 1 through W^T
    for (int l = P.p - 1; l >= 1; --l) {
      hm::HssLevelParams hp{W, B, xh, yh, l, k, nrhs, 0};
      int64_t total = ((int64_t)1 << l) * k * nrhs;
      unsigned blocks = (unsigned)std::min<int64_t>((total + hm::kThreads - 1) / hm::kThreads, 148 * 16);
      int slot = prof_begin("hss_up_level", stream);
      hm::hss_up_level_kernel<<<blocks, hm::kThreads, 0, stream>>>(hp);
      prof_end(slot, stream);
      ++g_launches;
      if ((st = cuda_check("hss_up_level_kernel"))) return st;
    }
    // Steps 2+3: coupling on level l (cores of the parents) + downsweep from l-1
    for (int l = 1; l <= P.p; ++l) {
      hm::HssLevelParams hp{R, B, xh, yh, l, k, nrhs, 0};
      int64_t total = ((int64_t)1 << l) * k * nrhs;
      unsigned blocks = (unsigned)std::min<int64_t>((total + hm::kThreads - 1) / hm::kThreads, 148 * 16);
      int slot = prof_begin("hss_down_level", stream);
      hm::hss_down_level_kernel<<<blocks, hm::kThreads, 0, stream>>>(hp);
      prof_end(slot, stream);
      ++g_launches;
      if ((st = cuda_check("hss_down_level_kernel"))) return st;
    }
  }
  // Step 4: Y(I_i) = U_i y_i^p + D_i X(I_i)
  hm::LeafParams lp;
  memset(&lp, 0, sizeof lp);
  lp.D = D; lp.X = Xd; lp.Y = Yd; lp.b = P.b; lp.m = nrhs; lp.mc = P.mc_leaf;
  if (coupled) {
    hm::LeafSeg& sg = lp.seg[lp.nseg++];
    sg.A = U;
    sg.T = yh + (((int64_t)1 << P.p) - 2) * k * nrhs;
    sg.k = k; sg.shift = 0; sg.xr = 0;
    lp.ktot = k;
  }
  if ((st = leaf_apply(lp, 1ll << P.p, P.mc_leaf, stream))) return st;
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
