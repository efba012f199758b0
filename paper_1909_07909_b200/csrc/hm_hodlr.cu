// hm_hodlr.cu — the HODLR product Y = A X (and A^T X) on the balanced tree:
// planning, the two phases (all levels' V^T X, then the leaf pass that adds
// D_i X(I_i) and every level's U_l t_l), the distributed phases
// and their C-ABI. Paper: Fig. 5 left, Def. 2.2,
// class P:226-235; O(k n log n).
#include "hm_internal.cuh"

namespace hmi {

// Row tile of the many-right-hand-side V^T X (vt_lv_kernel, one CTA per SM): 8
// leaves, or 4 when that fills the last wave of CTAs better — config 3 (512
// 8-leaf tiles on 148 SMs: 3.46 waves, the last one 46% full) runs 1024 4-leaf
// tiles (6.92 waves). Levels whose nodes span more than a tile reduce partials.
int64_t lv_tile(int64_t n, int64_t b) {
  const int64_t sms = num_sms();
  auto eff = [&](int64_t tile) {
    const int64_t t = n / tile;
    return (double)t / (double)(((t + sms - 1) / sms) * sms);
  };
  if (n % (8 * b) != 0) return 4 * b;
  return eff(4 * b) > eff(8 * b) + 0.02 ? 4 * b : 8 * b;
}

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
    P->tile = (nrhs >= 2 && HM_VT_TILE4 && nrhs < HM_VT_LV_MIN_M) ? 4 * b : (nrhs >= 2 ? lv_tile(n, b) : 8 * b);
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
    P->tile = (HM_VT_TILE4 && nrhs < HM_VT_LV_MIN_M) ? 4 * b : lv_tile(n, b);
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
        rl.block_begin = rp.blocks;
        int lg = 0;
        if (rl.per_node >= 512 && rl.km % 32 != 0) {
          rl.mode = 2;  // a CTA per output
          rp.blocks += rl.nodes * rl.km;
        } else if (rl.km % 32 == 0) {
          // warps per 32 outputs: ~8+ partials per warp, at most the CTA's 8 warps
          while (lg < 3 && (1 << lg) < rl.per_node / 8) ++lg;
          rl.mode = 1;
          const int64_t slabs = rl.nodes * rl.km / 32, per_block = (hm::kThreads / 32) >> lg;
          rp.blocks += (slabs + per_block - 1) / per_block;
        } else {
          while (lg < 5 && (1 << lg) < rl.per_node / 4) ++lg;  // ~4+ partials per lane
          rl.mode = 0;
          rp.blocks += ((rl.nodes * rl.km << lg) + hm::kThreads - 1) / hm::kThreads;
        }
        rl.log2g = lg;
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
    const unsigned grid = (unsigned)rp.blocks;
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
                           bool dtrans = false, bool skip_top = false) {
  hm::LeafParams lp;
  memset(&lp, 0, sizeof lp);
  lp.D = D; lp.X = Xd; lp.Y = Yd; lp.b = P.b; lp.m = P.m; lp.mc = P.mc_leaf; lp.dtrans = dtrans ? 1 : 0;
  int64_t uoff = 0, toff = 0;
  for (int l = 1; l <= P.q + P.p; ++l) {
    const int k = ranks[l - 1];
    if (k > 0 && !(skip_top && l <= P.q)) {
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
  if ((st = hodlr_vt_phase(P, ranks, op ? U : V, Xd, w, 1, P.p, nullptr, stream))) return st;
  if ((st = hodlr_leaf_phase(P, ranks, D, op ? V : U, Xd, Yd, w, nullptr, stream, op != 0))) return st;
  if (flags & HM_WS_HOSTIO) {
    if (cudaMemcpyAsync(Y, Yd, xy_bytes, cudaMemcpyDeviceToHost, stream) != cudaSuccess)
      return cuda_check("D2H copy of Y");
  }
  return HM_OK;
}

// ---- distributed HODLR ----

hm_status hodlr_dist_plan(const hm_tree* tree, const int32_t* ranks, int32_t nrhs, const hm_part* part, int32_t flags,
                          HodlrPlan* P, DistPart* d) {
  hm_status st = check_tree(tree);
  if (st) return st;
  if ((st = check_part(tree, part, d))) return st;
  return hodlr_plan_ex(tree->n >> d->q, tree->leaf, tree->levels - d->q, d->q, ranks, nrhs, flags, P);
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


// ---- distributed HODLR: the exchange's consumers ----

// t_l for the q top levels from the gathered per-rank partials: the sum, in
// rank order, over the ranks under the sibling of this rank's level-l ancestor.
hm_status hodlr_dist_combine(const HodlrPlan& P, const DistPart& d, const int32_t* ranks, const double* gathered,
                             double* ttop, cudaStream_t s) {
  if (P.top_doubles <= 0) return HM_OK;
  hm::CombineParams cp;
  memset(&cp, 0, sizeof cp);
  cp.gathered = gathered; cp.out = ttop; cp.per_rank = P.top_doubles; cp.q = d.q; cp.rank = d.rank;
  int64_t off = 0;
  for (int l = 1; l <= d.q; ++l) {
    cp.lev_off[l] = off;
    off += (int64_t)ranks[l - 1] * P.m;
  }
  cp.lev_off[d.q + 1] = off;
  const unsigned grid = (unsigned)((P.top_doubles + hm::kThreads - 1) / hm::kThreads);
  return launch("dist_combine", s, [&] { hm::dist_combine_kernel<<<grid, hm::kThreads, 0, s>>>(cp); });
}

// Y(I_r) += sum_{l <= q} U_l(I_r) t_l after a leaf pass that left the top levels out.
hm_status hodlr_top_epilogue(const HodlrPlan& P, const int32_t* ranks, const double* U, const double* ttop,
                             double* Y, cudaStream_t s) {
  hm::TopEpilogueParams ep;
  memset(&ep, 0, sizeof ep);
  ep.Y = Y; ep.U = U; ep.T = ttop; ep.n = P.n; ep.m = P.m;
  int64_t uoff = 0;
  for (int l = 1; l <= P.q; ++l) {
    const int k = ranks[l - 1];
    if (k > 0) {
      ep.k[ep.nlev] = k;
      ep.uoff[ep.nlev] = uoff;
      ++ep.nlev;
      ep.ktot += k;
    }
    uoff += P.n * k;
  }
  if (ep.nlev == 0) return HM_OK;
  const size_t smem = sizeof(double) * (size_t)ep.ktot * P.m;
  const unsigned grid = (unsigned)((P.n * P.m + hm::kThreads - 1) / hm::kThreads);
  return launch("dist_top_epilogue", s,
                [&] { hm::dist_top_epilogue_kernel<<<grid, hm::kThreads, smem, s>>>(ep); });
}

// The one-call product overlaps the allgather with the subtree's V^T X and the
// leaf pass, then adds the top-level terms in an epilogue — when the epilogue's
// extra Y read + write (16 m bytes per row) is at most 3% of the algorithmic
// bytes per row, 8 (b + 2 sum_l k_l + 2 m) (config 5: 0.7%). Otherwise the
// top-level terms stay in the leaf pass, which then waits for the exchange
// (it still overlaps the subtree's V^T X).
bool hodlr_dist_overlap_leaf(const HodlrPlan& P) {
  const double per_row = 8.0 * ((double)P.b + 2.0 * (double)P.ktot + 2.0 * P.m);
  return P.top_doubles > 0 && 16.0 * P.m <= 0.03 * per_row && P.top_doubles * 8 <= 48 * 1024;
}

struct HodlrDistWs {
  size_t off_send, off_gath, total;
};

HodlrDistWs hodlr_dist_ws(const HodlrPlan& P, int32_t nranks) {
  HodlrDistWs W;
  size_t off = align_up(P.total);
  W.off_send = off;
  off = align_up(off + sizeof(double) * (size_t)P.top_doubles);
  W.off_gath = off;
  off = align_up(off + sizeof(double) * (size_t)P.top_doubles * (size_t)nranks);
  W.total = off;
  return W;
}

}  // namespace hmi

using namespace hmi;

extern "C" {

// The power method's products run through the same routing as hodlr_matvec /
// hodlr_matvec_t: per-level ranks the uniform-tree kernels cannot take go to
// the general-tree kernels (then, like those calls, not graph-capturable).
hm_status hm_hodlr_norm2_workspace_bytes(const hm_tree* tree, const int32_t* ranks, size_t* bytes) {
  if (!bytes) return fail(HM_ERR_INVALID_ARG, "bytes is NULL");
  size_t mv = 0;
  hm_status st = hm_hodlr_workspace_bytes(tree, ranks, 1, 0, &mv);
  if (st) return st;
  *bytes = norm_plan(mv, tree->n).total;
  return HM_OK;
}

hm_status hodlr_norm2_est(const hm_tree* tree, const int32_t* ranks, const double* D, const double* U,
                          const double* V, const double* x0, int32_t iters, double* est, void* workspace,
                          size_t workspace_bytes, void* stream) {
  HM_NVTX("hodlr_norm2_est");
  size_t mv = 0;
  hm_status st = hm_hodlr_workspace_bytes(tree, ranks, 1, 0, &mv);
  if (st) return st;
  const NormPlan N = norm_plan(mv, tree->n);
  if (!workspace || workspace_bytes < N.total)
    return fail(HM_ERR_WORKSPACE, "workspace %zu bytes < required %zu", workspace_bytes, N.total);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return power_norm2(tree->n, x0, iters, est, static_cast<char*>(workspace), N, s,
                     [&](int op, const double* x, double* y) {
                       return op ? hodlr_matvec_t(tree, ranks, D, U, V, x, 1, y, workspace, mv, stream)
                                 : hodlr_matvec(tree, ranks, D, U, V, x, 1, y, workspace, mv, stream);
                     });
}

hm_status hm_hodlr_workspace_bytes(const hm_tree* tree, const int32_t* ranks, int32_t nrhs, int32_t flags,
                                   size_t* bytes) {
  if (!bytes) return fail(HM_ERR_INVALID_ARG, "bytes is NULL");
  if (flags == 0 && hodlr_use_general(tree, ranks, nrhs, flags)) {
    // per-level ranks: the general-tree kernels on the uniform endpoints
    const std::vector<int64_t> c = uniform_endpoints(tree);
    return hodlr_gen_workspace(tree->n, tree->levels, c.data(), ranks, nrhs, bytes);
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
  HM_NVTX("hodlr_matvec");
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
  HM_NVTX("hodlr_matvec_hostio");
  return hodlr_run(tree, ranks, D, U, V, X_host, nrhs, Y_host, workspace, workspace_bytes,
                   static_cast<cudaStream_t>(stream), HM_WS_HOSTIO);
}

hm_status hodlr_matvec_t(const hm_tree* tree, const int32_t* ranks, const double* D, const double* U,
                         const double* V, const double* X, int32_t nrhs, double* Y, void* workspace,
                         size_t workspace_bytes, void* stream) {
  HM_NVTX("hodlr_matvec_t");
  if (hodlr_use_general(tree, ranks, nrhs, 0)) {
    const std::vector<int64_t> c = uniform_endpoints(tree);
    return hodlr_gen_run(tree->n, tree->levels, c.data(), ranks, 1, D, U, V, X, nrhs, Y, workspace, workspace_bytes,
                         static_cast<cudaStream_t>(stream));
  }
  return hodlr_run(tree, ranks, D, U, V, X, nrhs, Y, workspace, workspace_bytes,
                   static_cast<cudaStream_t>(stream), 0, 1);
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
  HM_NVTX("hodlr_matvec_dist_begin");
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
                                  const double* D_local, const double* U_local, const double* V_local,
                                  const double* X_local, int32_t nrhs, double* Y_local, void* workspace,
                                  size_t workspace_bytes, void* stream) {
  HM_NVTX("hodlr_matvec_dist_local");
  HodlrPlan P;
  DistPart d;
  hm_status st = hodlr_dist_plan(tree, ranks, nrhs, part, 0, &P, &d);
  if (st) return st;
  if (!workspace || workspace_bytes < P.total) return fail(HM_ERR_WORKSPACE, "workspace too small");
  if (!X_local || (P.k > 0 && !V_local)) return fail(HM_ERR_INVALID_ARG, "NULL V / X pointer");
  const bool leaf_now = hodlr_dist_overlap_leaf(P);
  if (leaf_now) {
    if (!D_local || !aligned16(D_local)) return fail(HM_ERR_INVALID_ARG, "D_local NULL or misaligned");
    if ((st = hodlr_check_ptrs(P, D_local, U_local, V_local, X_local, Y_local, workspace, workspace_bytes, 0)))
      return st;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(workspace);
  g_launches = 0;
  prof_new_call();
  if ((st = hodlr_vt_phase(P, ranks, V_local, X_local, w, P.q + 1, P.q + P.p, nullptr, s))) return st;
  if (leaf_now)  // the leaf pass without the top levels, ahead of the exchange's result
    return hodlr_leaf_phase(P, ranks, D_local, U_local, X_local, Y_local, w, nullptr, s, false, true);
  return HM_OK;
}

hm_status hodlr_matvec_dist_end(const hm_tree* tree, const int32_t* ranks, const hm_part* part,
                                const double* D_local, const double* U_local, const double* X_local, int32_t nrhs,
                                const double* gathered, double* Y_local, void* workspace, size_t workspace_bytes,
                                void* stream) {
  HM_NVTX("hodlr_matvec_dist_end");
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
  if ((st = hodlr_dist_combine(P, d, ranks, gathered, ttop, s))) return st;
  if (hodlr_dist_overlap_leaf(P)) return hodlr_top_epilogue(P, ranks, U_local, ttop, Y_local, s);
  return hodlr_leaf_phase(P, ranks, D_local, U_local, X_local, Y_local, w, ttop, s);
}

// One call, NCCL inside: rank r's partial V_l(I_r)^T X(I_r) for
// the q top levels, their allgather on the communicator's stream while the
// subtree's V^T X and (hodlr_dist_overlap_leaf) the leaf pass run, then the
// combine and the top-level terms.
hm_status hm_hodlr_dist_workspace_bytes(const hm_tree* tree, const int32_t* ranks, int32_t nrhs, int32_t nranks,
                                        size_t* bytes) {
  if (!bytes) return fail(HM_ERR_INVALID_ARG, "bytes is NULL");
  const hm_part part{nranks, 0};
  HodlrPlan P;
  DistPart d;
  hm_status st = hodlr_dist_plan(tree, ranks, nrhs, &part, 0, &P, &d);
  if (st) return st;
  *bytes = hodlr_dist_ws(P, nranks).total;
  return HM_OK;
}

hm_status hodlr_matvec_dist(hm_comm* comm, const hm_tree* tree, const int32_t* ranks, const double* D_local,
                            const double* U_local, const double* V_local, const double* X_local, int32_t nrhs,
                            double* Y_local, void* workspace, size_t workspace_bytes, void* stream) {
  HM_NVTX("hodlr_matvec_dist");
  int32_t nranks = 0, rank = 0;
  hm_status st = comm_check(comm, &nranks, &rank);
  if (st) return st;
  const hm_part part{nranks, rank};
  HodlrPlan P;
  DistPart d;
  if ((st = hodlr_dist_plan(tree, ranks, nrhs, &part, 0, &P, &d))) return st;
  const HodlrDistWs W = hodlr_dist_ws(P, nranks);
  if (!D_local || !aligned16(D_local)) return fail(HM_ERR_INVALID_ARG, "D_local NULL or misaligned");
  if ((st = hodlr_check_ptrs(P, D_local, U_local, V_local, X_local, Y_local, workspace, workspace_bytes, 0)))
    return st;
  if (workspace_bytes < W.total)
    return fail(HM_ERR_WORKSPACE, "workspace %zu bytes < required %zu", workspace_bytes, W.total);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(workspace);
  double* send = reinterpret_cast<double*>(w + W.off_send);
  double* gathered = reinterpret_cast<double*>(w + W.off_gath);
  double* ttop = reinterpret_cast<double*>(w + P.off_ttop);
  const int64_t top = P.top_doubles;
  g_launches = 0;
  prof_new_call();
  if ((st = hodlr_vt_phase(P, ranks, V_local, X_local, w, 1, P.q, send, s))) return st;
  if ((st = comm_allgather_start(comm, send, top, gathered, s))) return st;
  if ((st = hodlr_vt_phase(P, ranks, V_local, X_local, w, P.q + 1, P.q + P.p, nullptr, s))) return st;
  if (hodlr_dist_overlap_leaf(P)) {
    if ((st = hodlr_leaf_phase(P, ranks, D_local, U_local, X_local, Y_local, w, nullptr, s, false, true))) return st;
    if ((st = comm_allgather_wait(comm, top, s))) return st;
    if ((st = hodlr_dist_combine(P, d, ranks, gathered, ttop, s))) return st;
    return hodlr_top_epilogue(P, ranks, U_local, ttop, Y_local, s);
  }
  if ((st = comm_allgather_wait(comm, top, s))) return st;
  if ((st = hodlr_dist_combine(P, d, ranks, gathered, ttop, s))) return st;
  return hodlr_leaf_phase(P, ranks, D_local, U_local, X_local, Y_local, w, ttop, s);
}

}  // extern "C"
