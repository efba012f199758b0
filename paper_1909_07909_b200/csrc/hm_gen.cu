// hm_gen.cu — general cluster trees: the leaf endpoint
// vector c of P:560-565 (Def. 2.1, empty leaves allowed, Fig. 4) and
// per-level HODLR ranks. Host tables derived from c, chunked V^T X with
// fixed-order per-node sums, general leaf pass; HSS tree sweeps reuse the
// uniform kernels (hm_hss.cu).
#include "hm_internal.cuh"
#include "hm_general.cuh"

namespace hmi {

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
  std::vector<int32_t> vt_k;           // rank of each vt level
  std::vector<int32_t> vt_order;       // chunk execution order (by first row, then level)
  std::vector<int32_t> leaf_order;     // leaf execution order (largest first)
  size_t off_tab, off_lo, off_doff, off_chunks, off_cbeg, off_vorder, off_lorder;
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
  // execution orders: chunks of all levels sorted by first row (then level), so the
  // CTAs reading the same X rows run in the same wave; leaves by decreasing size
  G->vt_order.resize(G->chunks.size());
  for (size_t c = 0; c < G->chunks.size(); ++c) G->vt_order[c] = (int32_t)c;
  std::stable_sort(G->vt_order.begin(), G->vt_order.end(), [&](int32_t a, int32_t b) {
    return G->chunks[a].lo < G->chunks[b].lo;
  });
  const int64_t nl = (int64_t)G->doff.size();
  G->leaf_order.resize(nl);
  for (int64_t i = 0; i < nl; ++i) G->leaf_order[i] = (int32_t)i;
  std::stable_sort(G->leaf_order.begin(), G->leaf_order.end(), [&](int32_t a, int32_t b) {
    return G->lo[a + 1] - G->lo[a] > G->lo[b + 1] - G->lo[b];
  });
  G->off_vorder = o; o = align_up(o + sizeof(int32_t) * G->vt_order.size());
  G->off_lorder = o; o = align_up(o + sizeof(int32_t) * G->leaf_order.size());
  G->tab_bytes = o;
  *off = align_up(*off + o);
  G->nchunks = (int64_t)G->chunks.size();
}

// Host image of the tables (built once per cached plan, see gen_cached).
void gen_build_image(const GenPlan& G, std::vector<char>* img) {
  img->assign(G.tab_bytes, 0);
  memcpy(img->data() + G.off_lo, G.lo.data(), sizeof(int64_t) * G.lo.size());
  memcpy(img->data() + G.off_doff, G.doff.data(), sizeof(int64_t) * G.doff.size());
  memcpy(img->data() + G.off_chunks, G.chunks.data(), sizeof(hm::GenChunk) * G.chunks.size());
  memcpy(img->data() + G.off_cbeg, G.cbeg.data(), sizeof(int64_t) * G.cbeg.size());
  memcpy(img->data() + G.off_vorder, G.vt_order.data(), sizeof(int32_t) * G.vt_order.size());
  memcpy(img->data() + G.off_lorder, G.leaf_order.data(), sizeof(int32_t) * G.leaf_order.size());
}

// The tables go to the workspace with one asynchronous copy from the plan's
// pinned image (PinnedImage: pinned once per cached plan), so the call neither
// synchronises the stream nor allocates.
hm_status gen_upload_tables(const PinnedImage& img, size_t off_tab, char* w, cudaStream_t s) {
  if (img.empty()) return HM_OK;
  if (!img.pinned) {
    if (cudaHostAlloc(reinterpret_cast<void**>(&img.pinned), img.size(), cudaHostAllocDefault) != cudaSuccess) {
      img.pinned = nullptr;
      return cuda_check("pinned copy of the tree tables");
    }
    memcpy(img.pinned, img.host.data(), img.size());
    if (cudaEventCreateWithFlags(&img.done, cudaEventDisableTiming) != cudaSuccess)
      return cuda_check("table upload event");
  }
  if (cudaMemcpyAsync(w + off_tab, img.pinned, img.size(), cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaEventRecord(img.done, s) != cudaSuccess)
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
  // 8 NT columns per CTA: NT = 1 up to 8 columns (no DMMAs on padding columns; ncu, ragged config-3 tree at
  // m = 8 with NT = 2: tensor pipe 48% busy, half of it on zero columns)
  if (k == 16) {
    if (vp.m <= 8) return gen_vt_mma_launch<16, 1>(vp, nchunks, s);
    return vp.m <= 16 ? gen_vt_mma_launch<16, 2>(vp, nchunks, s) : gen_vt_mma_launch<16, 4>(vp, nchunks, s);
  }
  if (k == 32) {
    if (vp.m <= 8) return gen_vt_mma_launch<32, 1>(vp, nchunks, s);
    return vp.m <= 16 ? gen_vt_mma_launch<32, 2>(vp, nchunks, s) : gen_vt_mma_launch<32, 4>(vp, nchunks, s);
  }
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
  vp.order = reinterpret_cast<const int32_t*>(w + G.off_tab + G.off_vorder);
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
  // Z rows, then the U segments' extended-column tables (pointer + stride per rank column)
  const size_t smem = sizeof(double) * (size_t)((smax + lp.ktot) * hm::gen_leaf_zs(MC)) + 16 * (size_t)lp.ktot + 16;
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
  if constexpr (!DT) {  // 128-bit A fragments (hm_general.cuh gen_leaf_mma_al_kernel)
    const size_t smem =
        sizeof(double) * (size_t)((smax + lp.ktot) * hm::gen_al_zs(NT)) + hm::gen_al_tab_bytes(lp.ktot);
    allow_smem(hm::gen_leaf_mma_al_kernel<NT>, smem);
    dim3 grid((unsigned)nleaves, (unsigned)((lp.m + NT * 8 - 1) / (NT * 8)));
    return launch("gen_leaf_mma", s, [&] { hm::gen_leaf_mma_al_kernel<NT><<<grid, hm::kThreads, smem, s>>>(lp); });
  }
  const size_t smem = sizeof(double) * (size_t)((smax + lp.ktot) * (NT * 8 + 4)) + 16 * (size_t)lp.ktot + 16;
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
    if (ranks[l - 1] > 0) {
      gen_add_vt_level(G, l);
      G->vt_k.push_back(ranks[l - 1]);
    }
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

hm_status hss_gen_plan(int64_t n, int32_t p, const int64_t* c, int32_t k, int32_t nrhs, GenPlan* G, HssPlan* H);

// Per-thread cache of the last few plans (key: the call's tree, ranks and nrhs,
// compared in full): repeated calls on one tree skip the host-side planning
// (chunk tables, sorts) and the image build.
struct GenCached {
  int kind;  // 0 HODLR, 1 HSS
  int64_t n;
  int32_t p, k, nrhs;
  std::vector<int64_t> c;
  std::vector<int32_t> ranks;
  GenPlan G;
  HssPlan H;
  PinnedImage img;
};

const GenCached* gen_cached(int kind, int64_t n, int32_t p, const int64_t* c, const int32_t* ranks, int32_t k,
                            int32_t nrhs, hm_status* st) {
  thread_local std::vector<GenCached> cache;  // most recent first
  const size_t nl = (p >= 0 && p <= 30) ? ((size_t)1 << p) : 0;
  const size_t nr = (kind == 0 && p > 0 && ranks) ? (size_t)p : 0;
  for (size_t e = 0; e < cache.size(); ++e) {
    const GenCached& g = cache[e];
    if (g.kind == kind && g.n == n && g.p == p && g.k == k && g.nrhs == nrhs && c && g.c.size() == nl &&
        memcmp(g.c.data(), c, nl * sizeof(int64_t)) == 0 && g.ranks.size() == nr &&
        (nr == 0 || memcmp(g.ranks.data(), ranks, nr * sizeof(int32_t)) == 0)) {
      if (e) std::rotate(cache.begin(), cache.begin() + e, cache.begin() + e + 1);
      *st = HM_OK;
      return &cache.front();
    }
  }
  GenCached g;
  g.kind = kind; g.n = n; g.p = p; g.k = k; g.nrhs = nrhs;
  *st = kind == 0 ? hodlr_gen_plan(n, p, c, ranks, nrhs, &g.G) : hss_gen_plan(n, p, c, k, nrhs, &g.G, &g.H);
  if (*st) return nullptr;
  g.c.assign(c, c + nl);
  if (nr) g.ranks.assign(ranks, ranks + nr);
  gen_build_image(g.G, &g.img.host);
  cache.insert(cache.begin(), std::move(g));
  if (cache.size() > 4) cache.pop_back();
  return &cache.front();
}

hm_status hodlr_gen_run(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks, int op, const double* D,
                        const double* U, const double* V, const double* X, int32_t nrhs, double* Y, void* ws,
                        size_t ws_bytes, cudaStream_t s) {
  hm_status st;
  const GenCached* gc = gen_cached(0, n, p, c, ranks, 0, nrhs, &st);
  if (st) return st;
  const GenPlan& G = gc->G;
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
  if ((st = gen_upload_tables(gc->img, G.off_tab, w, s))) return st;
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
  lp.order = reinterpret_cast<const int32_t*>(w + G.off_tab + G.off_lorder);
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
  if (coupled) {
    gen_add_vt_level(G, p);
    G->vt_k.push_back(k);
  }
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
  hm_status st;
  const GenCached* gc = gen_cached(1, n, p, c, nullptr, k, nrhs, &st);
  if (st) return st;
  const GenPlan& G = gc->G;
  const HssPlan& H = gc->H;
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
  if ((st = gen_upload_tables(gc->img, G.off_tab, w, s))) return st;
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
  lp.order = reinterpret_cast<const int32_t*>(w + G.off_tab + G.off_lorder);
  lp.doff = reinterpret_cast<const int64_t*>(w + G.off_tab + G.off_doff);
  if (coupled) {
    hm::LeafSeg& sg = lp.seg[lp.nseg++];
    sg.A = U; sg.T = yleaf; sg.k = k; sg.shift = 0; sg.xr = 0;
    lp.ktot = k;
  }
  return gen_leaf_phase(G, lp, s);
}

hm_status hodlr_gen_workspace(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks, int32_t nrhs,
                              size_t* bytes) {
  hm_status st;
  const GenCached* gc = gen_cached(0, n, p, c, ranks, 0, nrhs, &st);
  if (st) return st;
  *bytes = gc->G.total;
  return HM_OK;
}

}  // namespace hmi

using namespace hmi;

extern "C" {

// ---------------------------------------------------- general trees (f4) --

hm_status hm_hodlr_general_workspace_bytes(int64_t n, int32_t levels, const int64_t* c, const int32_t* ranks,
                                           int32_t nrhs, size_t* bytes) {
  if (!bytes) return fail(HM_ERR_INVALID_ARG, "bytes is NULL");
  return hodlr_gen_workspace(n, levels, c, ranks, nrhs, bytes);
}

hm_status hodlr_matvec_general(int64_t n, int32_t levels, const int64_t* c, const int32_t* ranks, int32_t op,
                               const double* D, const double* U, const double* V, const double* X, int32_t nrhs,
                               double* Y, void* workspace, size_t workspace_bytes, void* stream) {
  HM_NVTX("hodlr_matvec_general");
  if (op != 0 && op != 1) return fail(HM_ERR_INVALID_ARG, "op = %d (0: A X, 1: A^T X)", op);
  return hodlr_gen_run(n, levels, c, ranks, op, D, U, V, X, nrhs, Y, workspace, workspace_bytes,
                       static_cast<cudaStream_t>(stream));
}

hm_status hm_hss_general_workspace_bytes(int64_t n, int32_t levels, const int64_t* c, int32_t k, int32_t nrhs,
                                         size_t* bytes) {
  if (!bytes) return fail(HM_ERR_INVALID_ARG, "bytes is NULL");
  hm_status st;
  const GenCached* gc = gen_cached(1, n, levels, c, nullptr, k, nrhs, &st);
  if (st) return st;
  *bytes = gc->G.total;
  return HM_OK;
}

hm_status hss_matvec_general(int64_t n, int32_t levels, const int64_t* c, int32_t k, int32_t op, const double* D,
                             const double* U, const double* V, const double* R, const double* W, const double* B,
                             const double* X, int32_t nrhs, double* Y, void* workspace, size_t workspace_bytes,
                             void* stream) {
  HM_NVTX("hss_matvec_general");
  if (op != 0 && op != 1) return fail(HM_ERR_INVALID_ARG, "op = %d (0: A X, 1: A^T X)", op);
  return hss_gen_run(n, levels, c, k, op, D, U, V, R, W, B, X, nrhs, Y, workspace, workspace_bytes,
                     static_cast<cudaStream_t>(stream));
}

}  // extern "C"
