// hm_hss.cu — the HSS product Y = A X (and A^T X): planning, Step 1 (leaf
// V^T X + upsweep through W^T), Steps 2-3 (cores on every level l = 1..p,
// reading G1, and the downsweep through R), Step 4 (U_i y_i + D_i X(I_i)),
// the one-launch small-tree path, the distributed phases and
// their C-ABI. Paper: Fig. 5 right, eq. (3), class
// P:332-344; O(k n).
#include "hm_internal.cuh"
#include "hm_small.cuh"
#include "hm_tree.cuh"
#include "hm_treegemv.cuh"

// Trace names carry the column-tile count of the instance that ran (tests
// assert which instances a shape exercises): "<nt1>" = 8 columns per tile group.
#define HM_NT_NAME(base) (NT == 1 ? base "<nt1>" : NT == 2 ? base "<nt2>" : base "<nt4>")
#define HM_MB_NAME(base) (MB == 1 ? base "<m1>" : MB == 2 ? base "<m2>" : base "<m4>")

namespace hmi {

#ifndef HM_TREE_GEMV_MAXM
#define HM_TREE_GEMV_MAXM 1  // m = 2..4: the DMMA tree levels measured faster (C4 m=2: 490 vs 560 us)
#endif
constexpr int kTreeGemvMaxM = HM_TREE_GEMV_MAXM;
// One right-hand side (leaf 64 / 128 / 256, k in {16, 32, 64}): the DMMA path on
// one padded 8-column tile beats the GEMV kernels at every depth measured
// (tools/kbench.py hs:..., GEMV vs DMMA path: config 4 1461 vs 1295 us; p = 14
// leaf 64 k 16 / 32 / 64: 461 / 636 / 1370 vs 296 / 412 / 968 us; p = 12: 285 vs
// 245; p = 10: 152 vs 106; p = 8: 93 vs 59; p = 5: 37 vs 26 us — the warp-per-node
// down levels stream R, B at 3.7 TB/s, the dataflow launch halves the small
// levels). Minimum subtree depth for it; 0: off (the GEMV path).
#ifndef HM_M1_MMA_MINP
#define HM_M1_MMA_MINP 1
#endif

hm_status hss_plan_ex(int64_t n, int64_t b, int32_t p, int32_t q, int32_t k, int32_t nrhs, int32_t flags, HssPlan* P) {
  if (nrhs < 1) return fail(HM_ERR_INVALID_ARG, "nrhs = %d < 1", nrhs);
  if (k < 0) return fail(HM_ERR_INVALID_ARG, "k = %d < 0", k);
  if (k > hm::kMaxRank) return fail(HM_ERR_UNSUPPORTED, "rank %d > %d", k, hm::kMaxRank);
  memset(P, 0, sizeof *P);
  P->n = n; P->b = b; P->p = p; P->q = q; P->m = nrhs; P->k = k;
  const bool coupled = (k > 0 && p + q > 0);
  const bool leaf_coupled = (k > 0 && (p > 0 || q > 0));
  const bool m1_mma = HM_M1_MMA_MINP > 0 && nrhs == 1 && coupled && p >= HM_M1_MMA_MINP &&
                      (b == 64 || b == 128 || b == 256) && pow2_rank(k, 16, 64);
  const bool wide = nrhs >= 2 || m1_mma;  // the DMMA kernels (8-column tiles, masked)
  if (!coupled) {
    P->vt = VtPath::kNone;
  } else if (!wide && p >= 3 && b % 64 == 0 && b <= 4096 && pow2_rank(k, 1, 64)) {
    P->vt = VtPath::kGemv;
    P->tile = 8 * b;
  } else if (wide && b % 4 == 0 && pow2_rank(k, 16, 64)) {
    P->vt = VtPath::kMma;  // batched: warps per leaf
    P->nt_vt = nt_for(nrhs, HM_VTB_NTMAX);
  } else {
    P->vt = VtPath::kGeneric;
    P->mc_vt = vt_mc(b, nrhs);
    P->tile = pick_tile(b, p, P->mc_vt);
  }
  P->mma_levels = coupled && wide && pow2_rank(k, 16, 64);
  P->gemv_levels = coupled && !m1_mma && nrhs <= kTreeGemvMaxM && pow2_rank(k, 16, 64);
  if (P->mma_levels) P->nt_down = nt_for(nrhs, HM_TREE_NTMAX);
  const int ktot = leaf_coupled ? k : 0;
  if (!wide && b % 64 == 0 && b <= 1024 && (ktot == 0 || pow2_rank(ktot, 1, 64))) {
    P->leaf = LeafPath::kGemv;
  } else if (wide && (b == 64 || b == 128 || b == 256) && ktot % 8 == 0) {
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
  P->off_flags = off;  // dataflow tree kernel: ticket + per-pair flags (hss_tree_flow_kernel)
  if (P->mma_levels) off = align_up(off + sizeof(unsigned) * (size_t)(1 + (2ll << std::max(p, q))));
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
// Big upsweep levels with the pair's W staged in shared memory too
// (hss_up_stage; config 4: 238 vs 276 us for levels 14..11). The staged down
// kernel (hss_down_stage) measured slower there (469 vs 428 us: 67 KB per CTA,
// 3 CTAs per SM) and stays off; 0: the register-streaming pair kernels.
#ifndef HM_TREE_STAGE
#define HM_TREE_STAGE 1
#endif
#ifndef HM_TREE_STAGE_DOWN
#define HM_TREE_STAGE_DOWN 0
#endif
#ifndef HM_TREE_DOWN2
#define HM_TREE_DOWN2 1  // two big downsweep levels per launch (hss_down_two_kernel)
#endif
#ifndef HM_TREE_DOWN2_NT4
#define HM_TREE_DOWN2_NT4 1
#endif
#ifndef HM_TREE_DOWN2_MINB
#define HM_TREE_DOWN2_MINB 3  // measured: 2 -> 3 CTAs per SM, config 4 nrhs 16 down levels 153 -> 135 us
#endif


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
    st = launch(HM_MB_NAME("hss_up_gemv"), s, [&] { hm::hss_up_gemv_kernel<K, MB><<<grid, 256, 0, s>>>(tp, l); });
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
    st = launch(HM_MB_NAME("hss_tree_gemv_sweep"), s, [&] {
      e = cudaLaunchCooperativeKernel((const void*)hm::hss_tree_gemv_sweep_kernel<K, MB>, grid, dim3(256), args, 0,
                                      s);
    });
    if (st == HM_OK && e != cudaSuccess) return fail(HM_ERR_CUDA, "hss_tree_gemv_sweep: %s", cudaGetErrorString(e));
    if (st) return st;
  }
  for (int l = std::max(lbig, 1); down && l <= down_last; ++l) {
    const unsigned grid = (unsigned)(((1ll << l) + 7) / 8);
    st = launch(HM_MB_NAME("hss_down_gemv"), s, [&] { hm::hss_down_gemv_kernel<K, MB><<<grid, 256, 0, s>>>(tp, l); });
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

// Dataflow tree kernel (hss_tree_flow_kernel): every level of both sweeps in
// one launch, pair tasks ordered by flags instead of grid barriers. 0: the
// per-level launches + cooperative sweep below.
#ifndef HM_TREE_FLOW
#define HM_TREE_FLOW 1
#endif
#ifndef HM_FLOW_LEVELS
#define HM_FLOW_LEVELS 10  // levels 1..10 in the dataflow launch, the levels below one launch each
#endif

template <int KT, int NT>
hm_status tree_flow_launch(const hm::TreeParams& tp, bool up, bool down, cudaStream_t s, int up_from,
                           int down_last, unsigned* flags) {
  const size_t smem = sizeof(double) * (size_t)hm::flow_smem_doubles(KT, tp.m, NT);
  static int64_t cap = -1;  // resident CTAs of the instance (queried once)
  if (cap < 0) {
    allow_smem(hm::hss_tree_flow_kernel<KT, NT>, 200 * 1024);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hm::hss_tree_flow_kernel<KT, NT>, 256, smem) !=
        cudaSuccess)
      return cuda_check("occupancy query (hss_tree_flow)");
    cap = (int64_t)std::max(per_sm, 1) * num_sms();
  }
  const int L = up ? std::max(up_from, 0) : 0, DL = down ? std::max(down_last, 0) : 0;
  const int64_t tasks = (L >= 1 ? (1ll << L) - 1 : 0) + (DL >= 1 ? (1ll << DL) - 1 : 0);
  if (tasks == 0) return HM_OK;
  const size_t fbytes = sizeof(unsigned) * (size_t)(1 + (1ll << L) + (1ll << DL));
  if (cudaMemsetAsync(flags, 0, fbytes, s) != cudaSuccess) return cuda_check("hss_tree_flow flags");
  hm::FlowParams fp{tp, flags, L, DL, nullptr};
  const unsigned grid = (unsigned)std::min<int64_t>(cap, tasks);
#if HM_FLOW_TRACE
  // development builds: per-task timestamps of the last launch to $HM_FLOW_TRACE_FILE
  static unsigned long long* tr = nullptr;
  static int64_t tr_cap = 0;
  if (tr_cap < tasks) {
    if (tr) cudaFree(tr);
    cudaMalloc(&tr, sizeof(unsigned long long) * 6 * (size_t)tasks);
    tr_cap = tasks;
  }
  fp.trace = tr;
#endif
  hm_status st = launch(HM_NT_NAME("hss_tree_flow"), s,
                        [&] { hm::hss_tree_flow_kernel<KT, NT><<<grid, 256, smem, s>>>(fp); });
#if HM_FLOW_TRACE
  if (st == HM_OK && getenv("HM_FLOW_TRACE_FILE")) {
    std::vector<unsigned long long> h(6 * (size_t)tasks);
    cudaStreamSynchronize(s);
    cudaMemcpy(h.data(), tr, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost);
    if (FILE* f = fopen(getenv("HM_FLOW_TRACE_FILE"), "wb")) {
      int32_t hdr[4] = {L, DL, (int32_t)grid, (int32_t)tasks};
      fwrite(hdr, sizeof hdr, 1, f);
      fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
      fclose(f);
    }
  }
#endif
  return st;
}

template <int KT, int NT>
hm_status tree_launch(const hm::TreeParams& tp, int p, bool up, bool down, cudaStream_t s, int up_from_l,
                      int down_last, unsigned* flags) {
  const bool flow = HM_TREE_FLOW && flags && sizeof(double) * (size_t)hm::flow_smem_doubles(KT, tp.m, NT) <= 200 * 1024;
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
  const size_t smem_up_st = sizeof(double) * (size_t)hm::tree_up_stage_doubles(KT, tp.m, NT);
  const size_t smem_dn_st = sizeof(double) * (size_t)hm::tree_down_stage_doubles(KT, tp.m, NT);
  static bool attrs = false;
  int sweep_blocks_per_sm = 0;
  if (!attrs) {
    allow_smem(hm::hss_up_pair_kernel<KT, NT, MINB_UP>, 200 * 1024);
    allow_smem(hm::hss_down_pair_kernel<KT, NT, MINB>, 200 * 1024);
    allow_smem(hm::hss_tree_sweep_kernel<KT, NT>, 200 * 1024);
    allow_smem(hm::hss_up_stage_kernel<KT, NT>, 200 * 1024);
    allow_smem(hm::hss_down_stage_kernel<KT, NT>, 200 * 1024);
    attrs = true;
  }
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&sweep_blocks_per_sm, hm::hss_tree_sweep_kernel<KT, NT>, 256,
                                                    smem) != cudaSuccess)
    return cuda_check("occupancy query (hss_tree_sweep)");
  int lbig = 1;  // first level with >= kTreeBigLevel nodes
  while (lbig <= p && (1ll << lbig) < kTreeBigLevel) ++lbig;
  if (flow) lbig = HM_FLOW_LEVELS + 1;
  hm_status st;
  // upsweep: big levels up_from_l .. lbig one launch each
  for (int l = up_from_l; up && l >= lbig; --l) {
    const unsigned pairs = (unsigned)(1ll << (l - 1));
    if (HM_TREE_STAGE && smem_up_st <= 200 * 1024) {
      st = launch(HM_NT_NAME("hss_up_stage"), s,
                  [&] { hm::hss_up_stage_kernel<KT, NT><<<pairs, 256, smem_up_st, s>>>(tp, l); });
    } else {
      st = launch(HM_NT_NAME("hss_up_pair"), s,
                  [&] { hm::hss_up_pair_kernel<KT, NT, MINB_UP><<<pairs, 256, smem, s>>>(tp, l); });
    }
    if (st) return st;
  }
  // small levels: up min(p-1, lbig-1) .. 1, down 1 .. min(p, lbig-1), in one
  // cooperative launch. (Tried: the top levels 1..6 in one 16-CTA cluster with
  // cluster barriers — 67 + 72 us vs 140 us for the single sweep on config 4:
  // a level's cost is its own dependent load / DMMA / store chain, ~5.6 us, not
  // the barrier.)
  const int up_from = up ? std::min(up_from_l, lbig - 1) : 0, down_to = down ? std::min(down_last, lbig - 1) : 0;
  if (flow && (up_from >= 1 || down_to >= 1)) {
    if ((st = tree_flow_launch<KT, NT>(tp, up_from >= 1, down_to >= 1, s, up_from, down_to, flags))) return st;
  } else if (up_from >= 1 || down_to >= 1) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t need = std::max<int64_t>(1, (1ll << std::max(up_from, down_to)) / 2);
    dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)sweep_blocks_per_sm * sms, need)));
    hm::TreeParams arg = tp;
    int a1 = up_from, a2 = 1, a3 = 1, a4 = down_to;
    void* args[] = {&arg, &a1, &a2, &a3, &a4};
    cudaError_t e = cudaSuccess;
    st = launch(HM_NT_NAME("hss_tree_sweep"), s, [&] {
      e = cudaLaunchCooperativeKernel((const void*)hm::hss_tree_sweep_kernel<KT, NT>, grid, dim3(256), args, smem, s);
    });
    if (st == HM_OK && e != cudaSuccess) return fail(HM_ERR_CUDA, "hss_tree_sweep: %s", cudaGetErrorString(e));
    if (st) return st;
  }
  // downsweep: big levels lbig .. p one launch each, or two per launch
  // (hss_down_two, pairs ending at down_last): up to 16 columns with 9 staged
  // blocks, 32 columns (one phase-A task per warp) with y_l over x_l (7 blocks);
  // 3 CTAs per SM (KT = 64: 2, 3 would spill)
  constexpr int MINB2 = KT >= 64 ? 2 : HM_TREE_DOWN2_MINB;
  const int ntask_a = (KT / 8) * (hm::tree_mpad(tp.m, NT) / (NT * 8));
  const bool alias = NT == 4 && ntask_a <= 4;
  const size_t smem_two = sizeof(double) * (size_t)hm::tree_down_two_doubles(KT, tp.m, NT, alias);
  const bool two_ok = HM_TREE_DOWN2 && (NT <= 2 || (alias && HM_TREE_DOWN2_NT4)) && smem_two <= 110 * 1024;
  if (two_ok) {
    if (alias) allow_smem(hm::hss_down_two_kernel<KT, NT, MINB2, true>, smem_two);
    else allow_smem(hm::hss_down_two_kernel<KT, NT, MINB2, false>, smem_two);
  }
  for (int l = std::max(lbig, 1); down && l <= down_last; ++l) {
    const unsigned pairs = (unsigned)(1ll << (l - 1));
    if (two_ok && l >= 2 && l + 1 <= down_last && (down_last - l + 1) % 2 == 0) {
      st = launch(HM_NT_NAME("hss_down_two"), s, [&] {
        if (alias) hm::hss_down_two_kernel<KT, NT, MINB2, true><<<pairs, 256, smem_two, s>>>(tp, l);
        else hm::hss_down_two_kernel<KT, NT, MINB2, false><<<pairs, 256, smem_two, s>>>(tp, l);
      });
      if (st) return st;
      ++l;
      continue;
    }
    if (HM_TREE_STAGE_DOWN && smem_dn_st <= 200 * 1024) {
      st = launch(HM_NT_NAME("hss_down_stage"), s,
                  [&] { hm::hss_down_stage_kernel<KT, NT><<<pairs, 256, smem_dn_st, s>>>(tp, l); });
    } else {
      st = launch(HM_NT_NAME("hss_down_pair"), s,
                  [&] { hm::hss_down_pair_kernel<KT, NT, MINB><<<pairs, 256, smem, s>>>(tp, l); });
    }
    if (st) return st;
  }
  return HM_OK;
}

hm_status tree_dispatch(const hm::TreeParams& tp, int p, int k, int nt, bool up, bool down, cudaStream_t s,
                        int up_from, int down_last, unsigned* flags) {
#define HM_TREE(KT_)                                                                        \
  if (k == KT_) {                                                                           \
    if (nt == 1) return tree_launch<KT_, 1>(tp, p, up, down, s, up_from, down_last, flags); \
    if (nt == 2) return tree_launch<KT_, 2>(tp, p, up, down, s, up_from, down_last, flags); \
    return tree_launch<KT_, 4>(tp, p, up, down, s, up_from, down_last, flags);              \
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
                         cudaStream_t stream, int bt, int up_from, int down_last, unsigned* flow_flags) {
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
    return tree_dispatch(tp, p, k, P.nt_down, up, down, stream, up_from, down_last, flow_flags);
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

// Step 1 on the subtree: leaf x = V^T X, upsweep to level 1, and (W_root given)
// the subtree root's x_root = W_root^T [x_{1,0}; x_{1,1}]. A depth-0 subtree is
// one leaf: its x is the root's, written to x_root.
// Step 1 fused with the first three upsweep levels (hss_vt_up_kernel): k in
// {16, 32}, nrhs <= 16, a tree of depth >= 4. Measured on config 4's tree
// (kbench c4 / c4m8): m = 8: 313 us vs 341 (vt_batched + the three up-pair
// launches); m = 32: 702 vs 622 — at two CTAs per SM the x-only phases 2-4
// leave the memory pipe idle, so m = 32 keeps the separate kernels.
#ifndef HM_VT_UP
#define HM_VT_UP 1
#endif
bool vt_up_ok(const HssPlan& P) {
  return HM_VT_UP && P.vt == VtPath::kMma && (P.k == 16 || P.k == 32) && P.m <= 16 && P.p >= 4 &&
         P.b % 4 == 0;
}

template <int KT, int NT>
hm_status vt_up_launch(const hm::VtUpParams& vp, int64_t ctas, cudaStream_t s) {
  const size_t smem = sizeof(double) * 12 * KT * (NT * 8 + 4);
  allow_smem(hm::hss_vt_up_kernel<KT, NT>, smem);
  return launch("hss_vt_up", s, [&] { hm::hss_vt_up_kernel<KT, NT><<<(unsigned)ctas, 256, smem, s>>>(vp); });
}

hm_status vt_up_dispatch(const HssPlan& P, const double* V, const double* W, const double* Xd, double* xh,
                         cudaStream_t s) {
  const hm::VtUpParams vp{V, Xd, W, xh, (int32_t)P.b, P.m, P.p};
  const int64_t ctas = ((int64_t)1 << P.p) / 8;
  const int nt = nt_for(P.m, 4);
#define HM_VU(KT_)                                                 if (P.k == KT_) {                                                  if (nt == 1) return vt_up_launch<KT_, 1>(vp, ctas, s);           if (nt == 2) return vt_up_launch<KT_, 2>(vp, ctas, s);           return vt_up_launch<KT_, 4>(vp, ctas, s);                      }
  HM_VU(16)
  HM_VU(32)
#undef HM_VU
  return fail(HM_ERR_UNSUPPORTED, "hss_vt_up: no instance for k=%d", P.k);
}

// up_from_out != NULL: the tree levels are left to the caller (one launch with
// the downsweep, hss_tree_flow_kernel), *up_from_out = the first level to compute.
hm_status hss_up_phase(const HssPlan& P, const double* V, const double* W, const double* Xd, double* xh,
                       const double* W_root, double* x_root, cudaStream_t stream, int* up_from_out = nullptr) {
  const int k = P.k, nrhs = P.m;
  const int64_t km = (int64_t)k * nrhs;
  hm_status st;
  double* xleaf = (P.p == 0) ? x_root : xh + (((int64_t)1 << P.p) - 2) * km;
  if (xleaf == nullptr) return HM_OK;
  int up_from = P.p - 1;
  if (vt_up_ok(P)) {
    // Step 1 + upsweep levels p-1, p-2, p-3 in one launch (hss_vt_up_kernel)
    if ((st = vt_up_dispatch(P, V, W, Xd, xh, stream))) return st;
    up_from = P.p - 4;
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
  if (up_from_out) {
    *up_from_out = up_from;
    return HM_OK;
  }
  if (up_from >= 1 && (st = hss_tree_phase(P, P.p, W, nullptr, nullptr, xh, nullptr, nullptr, nullptr, true,
                                             false, stream, 0, up_from)))
    return st;
  if (W_root && P.p >= 1 && (st = hss_single_vt(P, W_root, xh, 2 * k, x_root, stream))) return st;
  return HM_OK;
}

// Step 4: Y(I_i) = U_i y_i + D_i X(I_i); y of the leaves from yh (or y_root for a
// depth-0 subtree).
hm_status hss_leaf_phase(const HssPlan& P, const double* D, const double* U, const double* Xd, double* Yd,
                         const double* yleaf, cudaStream_t stream, bool dtrans = false) {
  hm::LeafParams lp;
  memset(&lp, 0, sizeof lp);
  lp.D = D; lp.X = Xd; lp.Y = Yd; lp.b = P.b; lp.m = P.m; lp.mc = P.mc_leaf; lp.dtrans = dtrans ? 1 : 0;
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

// HSS Step 4 with the leaf level's coupling + downsweep (hm_fast.cuh
// leaf_mma_down_kernel) instead of a separate level-p downsweep launch.
#ifndef HM_LEAF_DOWN
#define HM_LEAF_DOWN 1
#endif

// ---- small trees: one cooperative launch (hm_small.cuh) ----
#ifndef HM_NO_SMALL
#define HM_NO_SMALL 0
#endif
// One CTA per leaf streams its D_i alone, so the launch pays off only while the
// leaves are few or small: depth <= 6, or 7 with 64-row leaves. Measured against
// the level-by-level DMMA path (tools/kbench.py hs:..., k = 32, one launch vs
// levels): p = 8 leaf 128, nrhs 1 / 2 / 8 / 16 / 32: 96 / 97 / 102 / 129 / 218 vs
// 59 / 57 / 54 / 66 / 109 us; p = 8 leaf 64, nrhs 1 / 2: 83 / 84 vs 52 / 48 us;
// p = 7 leaf 128, nrhs 1 / 2 / 8 / 16 / 32: 61 / 60 / 66 / 73 / 116 vs 50 / 47 /
// 48 / 54 / 89 us; p = 7 leaf 64 (k 16, nrhs 1): 28 vs 37 us; p = 6: 46 vs 45,
// 39 vs 40 us; p = 5: 26 vs 33 us; p <= 4: 18-30 vs 25-32 us.
// HM_SMALL_DEEP_ALL 0: the depth rule at nrhs 1 only (nrhs >= 2 up to depth 8).
#ifndef HM_SMALL_DEEP_ALL
#define HM_SMALL_DEEP_ALL 1
#endif
constexpr int kSmallMaxLevels = 8;  // up to 256 leaves: one CTA per leaf, all co-resident

bool small_ok(const HssPlan& P) {
  if (HM_NO_SMALL || P.q != 0 || !P.mma_levels || P.p < 1 || P.p > kSmallMaxLevels || P.m > 32 ||
      !(P.b == 64 || P.b == 128))
    return false;
  if (P.m == 1 || HM_SMALL_DEEP_ALL) return P.p <= 6 || (P.p == 7 && P.b == 64);
  return true;
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
  // the leaf level's coupling + downsweep inside the leaf pass (leaf_mma_down_kernel)
  // for up to 16 columns per CTA: measured on config 4's tree, nrhs 8 / 16: 1473 ->
  // 1439 / 1744 -> 1703 us; at 32 columns the leaf pass sits at the fp64 ridge and
  // the extra DMMAs cost more than the separate HBM-bound launch (2465 -> 2550 us)
  const bool fuse_down = HM_LEAF_DOWN && coupled && op == 0 && P.mma_levels && !P.gemv_levels &&
                         P.leaf == LeafPath::kMma && P.p >= 2 && P.nt_leaf <= 2 &&
                         leaf_down_supported(P.b, k, P.nt_leaf);
  if (coupled) {
    // Step 1 (leaf x), then the upsweep levels and Steps 2-3 in one tree phase
    int up_from = 0;
    if ((st = hss_up_phase(P, V, W, Xd, xh, nullptr, nullptr, stream, &up_from))) return st;
    unsigned* fl = reinterpret_cast<unsigned*>(w + P.off_flags);
    if ((st = hss_tree_phase(P, P.p, W, R, B, xh, yh, nullptr, nullptr, up_from >= 1, true, stream, op,
                             std::max(up_from, 1), fuse_down ? P.p - 1 : -1, P.mma_levels ? fl : nullptr)))
      return st;
  }
  const double* yleaf = coupled ? yh + (((int64_t)1 << P.p) - 2) * km : nullptr;
  if (fuse_down) {
    hm::LeafParams lp;
    memset(&lp, 0, sizeof lp);
    lp.D = D; lp.X = Xd; lp.Y = Yd; lp.b = P.b; lp.m = P.m; lp.mc = P.mc_leaf;
    hm::LeafSeg& sg = lp.seg[lp.nseg++];
    sg.A = U; sg.T = yleaf; sg.k = k; sg.shift = 0; sg.xr = 0;
    lp.ktot = k;
    const hm::LeafDownParams q{B, R, xh + (((int64_t)1 << P.p) - 2) * km, yh + (((int64_t)1 << (P.p - 1)) - 2) * km,
                               P.p, 0};
    st = leaf_down_dispatch(lp, q, 1ll << P.p, k, P.nt_leaf, stream);
    if (st == HM_ERR_UNSUPPORTED) return fail(HM_ERR_UNSUPPORTED, "leaf_mma_down: no instance (b=%lld, nt=%d)",
                                              (long long)P.b, P.nt_leaf);
    if (st) return st;
  } else if ((st = hss_leaf_phase(P, D, U, Xd, Yd, yleaf, stream, op != 0))) {
    return st;
  }
  if (flags & HM_WS_HOSTIO) {
    if (cudaMemcpyAsync(Y, Yd, xy_bytes, cudaMemcpyDeviceToHost, stream) != cudaSuccess)
      return cuda_check("D2H copy of Y");
  }
  return HM_OK;
}

// ---- per-level ranks ----
//
// k_l = ranks[l-1] columns on level l: U, V [n][k_p]; R, W of node (l, i)
// [2k_{l+1}][k_l]; the cores of the level-l siblings [2][k_l][k_l] (include/hm.h
// hss_matvec_ranked has the offsets). Step 1 and Step 4 run the uniform leaf
// kernels with k = k_p; the tree levels run hss_up_ranked / hss_down_ranked.
// Equal ranks take hss_run (the tuned tree kernels).
struct RankedPlan {
  HssPlan P;  // leaf-level paths for k_p
  int32_t kl[hm::kMaxLevels + 2];
  int64_t cf[hm::kMaxLevels + 2], rw[hm::kMaxLevels + 2], bo[hm::kMaxLevels + 2];
  size_t off_xh, off_yh, total;
  bool uniform;
};

// DMMA level kernels (hm_tree.cuh) when the output rank is a multiple of 8 and
// the contraction lengths multiples of 4; otherwise the CUDA-core ones.
#ifndef HM_RANKED_MMA
#define HM_RANKED_MMA 1
#endif
#ifndef HM_RANKED_MMA_MINM
#define HM_RANKED_MMA_MINM 1  // nrhs 1 too (one masked column tile): per-level HSS, 13 levels, nrhs 1: 508 -> 347 us
#endif
bool ranked_mma_ok(int k, int kin, int kp, int32_t nrhs) {
  return HM_RANKED_MMA && nrhs >= HM_RANKED_MMA_MINM && k % 8 == 0 && kin % 4 == 0 && kp % 4 == 0;
}

template <int NT>
hm_status ranked_mma_launch_nt(const hm::RankedMmaParams& rp, bool up, cudaStream_t s) {
  const int64_t warps = rp.nodes * (rp.k / 8) * ((rp.m + NT * 8 - 1) / (NT * 8));
  const unsigned grid = (unsigned)((warps + 7) / 8);
  if (up)
    return launch(HM_NT_NAME("hss_up_ranked_mma"), s,
                  [&] { hm::hss_up_ranked_mma_kernel<NT><<<grid, 256, 0, s>>>(rp); });
  return launch(HM_NT_NAME("hss_down_ranked_mma"), s,
                [&] { hm::hss_down_ranked_mma_kernel<NT><<<grid, 256, 0, s>>>(rp); });
}

hm_status ranked_mma_launch(const hm::RankedMmaParams& rp, bool up, cudaStream_t s) {
  if (rp.m <= 8) return ranked_mma_launch_nt<1>(rp, up, s);
  if (rp.m <= 16) return ranked_mma_launch_nt<2>(rp, up, s);
  return ranked_mma_launch_nt<4>(rp, up, s);
}

// The small levels (< kRankedSweepNodes nodes) of both per-level-rank sweeps in
// one cooperative launch (hss_ranked_sweep_kernel): a grid barrier between
// levels instead of a kernel boundary.
#ifndef HM_RANKED_SWEEP
#define HM_RANKED_SWEEP 1
#endif
constexpr int64_t kRankedSweepNodes = 2048;

template <int NT, typename Steps>
hm_status ranked_sweep_launch_nt(const Steps& steps, size_t w0, size_t w1, cudaStream_t s) {
  static int per_sm = -1, sms = 0;
  if (per_sm < 0) {
    int dev = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hm::hss_ranked_sweep_kernel<NT>, 256, 0) !=
        cudaSuccess)
      return cuda_check("occupancy query (hss_ranked_sweep)");
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  hm::RankedSweepParams sp;
  memset(&sp, 0, sizeof sp);
  int64_t most = 1;
  for (size_t i = w0; i < w1; ++i) {
    sp.step[sp.nsteps] = steps[i].rp;
    sp.up[sp.nsteps] = steps[i].up ? 1 : 0;
    ++sp.nsteps;
    most = std::max<int64_t>(most, steps[i].rp.nodes * (steps[i].rp.k / 8) * ((steps[i].rp.m + NT * 8 - 1) / (NT * 8)));
  }
  dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * sms, (most + 7) / 8)));
  void* args[] = {&sp};
  cudaError_t e = cudaSuccess;
  hm_status st = launch(HM_NT_NAME("hss_ranked_sweep"), s, [&] {
    e = cudaLaunchCooperativeKernel((const void*)hm::hss_ranked_sweep_kernel<NT>, grid, dim3(256), args, 0, s);
  });
  if (st == HM_OK && e != cudaSuccess) return fail(HM_ERR_CUDA, "hss_ranked_sweep: %s", cudaGetErrorString(e));
  return st;
}

template <typename Steps>
hm_status ranked_sweep_launch(const Steps& steps, size_t w0, size_t w1, int32_t m, cudaStream_t s) {
  if (m <= 8) return ranked_sweep_launch_nt<1>(steps, w0, w1, s);
  if (m <= 16) return ranked_sweep_launch_nt<2>(steps, w0, w1, s);
  return ranked_sweep_launch_nt<4>(steps, w0, w1, s);
}

hm_status hss_ranked_plan(const hm_tree* tree, const int32_t* ranks, int32_t nrhs, RankedPlan* Q) {
  hm_status st = check_tree(tree);
  if (st) return st;
  memset(Q, 0, sizeof *Q);
  const int p = tree->levels;
  if (p > 0 && !ranks) return fail(HM_ERR_INVALID_ARG, "ranks is NULL");
  if (nrhs < 1) return fail(HM_ERR_INVALID_ARG, "nrhs = %d < 1", nrhs);
  Q->uniform = true;
  for (int l = 1; l <= p; ++l) {
    const int k = ranks[l - 1];
    if (k < 0) return fail(HM_ERR_INVALID_ARG, "ranks[%d] = %d < 0", l - 1, k);
    if (k > hm::kMaxRank) return fail(HM_ERR_UNSUPPORTED, "rank %d > %d", k, hm::kMaxRank);
    Q->kl[l] = k;
    Q->uniform = Q->uniform && k == ranks[0];
  }
  const int kp = p > 0 ? Q->kl[p] : 0;
  if ((st = hss_plan_ex(tree->n, tree->leaf, p, 0, kp, nrhs, 0, &Q->P))) return st;
  for (int l = 1; l <= p; ++l) {
    Q->cf[l + 1] = Q->cf[l] + ((int64_t)1 << l) * Q->kl[l] * nrhs;
    Q->bo[l + 1] = Q->bo[l] + ((int64_t)1 << (l - 1)) * 2 * Q->kl[l] * Q->kl[l];
    if (l <= p - 1) Q->rw[l + 1] = Q->rw[l] + ((int64_t)1 << l) * 2 * Q->kl[l + 1] * Q->kl[l];
  }
  size_t off = 0;
  Q->off_xh = off;
  off = align_up(off + sizeof(double) * (size_t)Q->cf[p + 1]);
  Q->off_yh = off;
  off = align_up(off + sizeof(double) * (size_t)Q->cf[p + 1]);
  Q->total = std::max<size_t>(off, kAlign);
  if (Q->uniform) {  // the tuned path's own workspace
    HssPlan U;
    if ((st = hss_plan(tree, p > 0 ? ranks[0] : 0, nrhs, 0, &U))) return st;
    Q->total = std::max(Q->total, U.total);
  }
  return HM_OK;
}

hm_status hss_ranked_run(const hm_tree* tree, const int32_t* ranks, int op, const double* D, const double* U,
                         const double* V, const double* R, const double* W, const double* B, const double* X,
                         int32_t nrhs, double* Y, void* ws, size_t ws_bytes, cudaStream_t s) {
  RankedPlan Q;
  hm_status st = hss_ranked_plan(tree, ranks, nrhs, &Q);
  if (st) return st;
  if (Q.uniform)
    return hss_run(tree, tree->levels > 0 ? ranks[0] : 0, D, U, V, R, W, B, X, nrhs, Y, ws, ws_bytes, s, 0, op);
  const HssPlan& P = Q.P;
  const int p = P.p;
  if (!D || !X || !Y) return fail(HM_ERR_INVALID_ARG, "NULL D / X / Y pointer");
  if (!aligned16(D) || !aligned16(X) || !aligned16(Y)) return fail(HM_ERR_INVALID_ARG, "D, X, Y must be 16-byte aligned");
  if (!ws || ws_bytes < Q.total || !aligned16(ws))
    return fail(HM_ERR_WORKSPACE, "workspace %zu bytes < required %zu (or misaligned)", ws_bytes, Q.total);
  const size_t xy = sizeof(double) * (size_t)(P.n * nrhs);
  if (overlap(X, xy, Y, xy)) return fail(HM_ERR_INVALID_ARG, "X and Y overlap");
  bool any = false, any_t = false, any_b = false;
  for (int l = 1; l <= p; ++l) {
    any = any || Q.kl[l] > 0;
    any_b = any_b || Q.kl[l] > 0;
    if (l <= p - 1) any_t = any_t || (Q.kl[l] > 0 && Q.kl[l + 1] > 0);
  }
  if ((Q.kl[p] > 0 && p > 0 && (!U || !V)) || (any_b && !B) || (any_t && (!R || !W)))
    return fail(HM_ERR_INVALID_ARG, "NULL generator pointer");
  if (op) {  // A^T: U <-> V, R <-> W, transposed cores, D_i^T
    std::swap(U, V);
    std::swap(R, W);
  }
  char* w = static_cast<char*>(ws);
  double* xh = reinterpret_cast<double*>(w + Q.off_xh);
  double* yh = reinterpret_cast<double*>(w + Q.off_yh);
  const int kp = p > 0 ? Q.kl[p] : 0;
  g_launches = 0;
  prof_new_call();
  auto grid_for = [](int64_t total) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((total + hm::kThreads - 1) / hm::kThreads, 148 * 16));
  };
  if (any) {
    // Step 1: x of the leaves, V_i^T X(I_i) with k_p columns (the uniform leaf-level kernels)
    if (kp > 0) {
      double* xleaf = xh + Q.cf[p];
      if (P.vt == VtPath::kMma) {
        hm::BatchedVtParams bp{V, P.b * kp, X, P.b * nrhs, xleaf, (int64_t)kp * nrhs, (int64_t)1 << p, (int32_t)P.b,
                               nrhs};
        if ((st = vt_batched_dispatch("vt_batched", bp, kp, P.nt_vt, s))) return st;
      } else {
        hm::VtParams vp;
        memset(&vp, 0, sizeof vp);
        vp.X = X; vp.n = P.n; vp.m = nrhs; vp.mc = P.mc_vt ? P.mc_vt : vt_mc(P.b, nrhs);
        vp.tile = P.tile ? P.tile : pick_tile(P.b, p, vp.mc); vp.nlev = 1;
        vp.lev[0].V = V; vp.lev[0].k = kp; vp.lev[0].s = P.b; vp.lev[0].out = xleaf; vp.lev[0].partial = nullptr;
        st = (P.vt == VtPath::kGemv) ? vt_gemv_dispatch(vp, P.b, kp, s) : vt_generic(vp, P.n, s);
        if (st) return st;
      }
    }
    // the level steps in execution order: upsweep l = p-1..1 through W^T
    // (2k_{l+1} x k_l), then cores (levels 1..p, reading G1) + downsweep through R
    struct Step {
      bool up, mma;
      int l;
      hm::RankedMmaParams rp;
      hm::HssRankedLevelParams hp;
    };
    std::vector<Step> steps;
    for (int l = p - 1; l >= 1; --l) {
      if (Q.kl[l] == 0) continue;
      Step t;
      t.up = true;
      t.l = l;
      t.mma = ranked_mma_ok(Q.kl[l], 2 * Q.kl[l + 1], 0, nrhs);
      t.rp = hm::RankedMmaParams{W + Q.rw[l], nullptr, xh + Q.cf[l + 1], nullptr, xh + Q.cf[l], (int64_t)1 << l,
                                 Q.kl[l], Q.kl[l + 1], 0, nrhs, 0};
      t.hp = hm::HssRankedLevelParams{W + Q.rw[l], nullptr, xh + Q.cf[l + 1], nullptr, xh + Q.cf[l], l, Q.kl[l],
                                      Q.kl[l + 1], 0, nrhs, 0};
      steps.push_back(t);
    }
    for (int l = 1; l <= p; ++l) {
      if (Q.kl[l] == 0) continue;
      const bool from_parent = l >= 2 && Q.kl[l - 1] > 0;
      Step t;
      t.up = false;
      t.l = l;
      t.mma = ranked_mma_ok(Q.kl[l], Q.kl[l], from_parent ? Q.kl[l - 1] : 0, nrhs);
      t.rp = hm::RankedMmaParams{from_parent ? R + Q.rw[l - 1] : nullptr, B + Q.bo[l], xh + Q.cf[l],
                                 from_parent ? yh + Q.cf[l - 1] : nullptr, yh + Q.cf[l], (int64_t)1 << l, Q.kl[l], 0,
                                 from_parent ? Q.kl[l - 1] : 0, nrhs, op};
      t.hp = hm::HssRankedLevelParams{from_parent ? R + Q.rw[l - 1] : nullptr, B + Q.bo[l], xh + Q.cf[l],
                                      from_parent ? yh + Q.cf[l - 1] : nullptr, yh + Q.cf[l], l, Q.kl[l], 0,
                                      from_parent ? Q.kl[l - 1] : 0, nrhs, op};
      steps.push_back(t);
    }
    // the small levels (contiguous in this order: the top of both sweeps) in one
    // cooperative launch when every one of them takes the DMMA kernels
    size_t w0 = steps.size(), w1 = steps.size();
    for (size_t i = 0; i < steps.size(); ++i)
      if (((int64_t)1 << steps[i].l) < kRankedSweepNodes) {
        w0 = std::min(w0, i);
        w1 = i + 1;
      }
    bool sweep = HM_RANKED_SWEEP && w1 > w0 + 1;
    for (size_t i = w0; sweep && i < w1; ++i) sweep = steps[i].mma;
    for (size_t i = 0; i < steps.size(); ++i) {
      if (sweep && i == w0) {
        if ((st = ranked_sweep_launch(steps, w0, w1, nrhs, s))) return st;
        i = w1 - 1;
        continue;
      }
      const Step& t = steps[i];
      if (t.mma) {
        if ((st = ranked_mma_launch(t.rp, t.up, s))) return st;
        continue;
      }
      const int64_t total = ((int64_t)1 << t.l) * Q.kl[t.l] * nrhs;
      const hm::HssRankedLevelParams hp = t.hp;
      st = t.up ? launch("hss_up_ranked", s,
                         [&] { hm::hss_up_ranked_kernel<<<grid_for(total), hm::kThreads, 0, s>>>(hp); })
                : launch("hss_down_ranked", s,
                         [&] { hm::hss_down_ranked_kernel<<<grid_for(total), hm::kThreads, 0, s>>>(hp); });
      if (st) return st;
    }
  }
  // Step 4: Y(I_i) = U_i y_i + D_i X(I_i) (k_p columns)
  const double* yleaf = (p > 0 && kp > 0) ? yh + Q.cf[p] : nullptr;
  return hss_leaf_phase(P, D, U, X, Y, yleaf, s, op != 0);
}

// ---- per-node ranks ----
//
// Node (l, i) has rank k_h, h = 2^l - 2 + i. The compact generators (layout
// of include/hm.h hss_matvec_noderanked) are zero-padded into the uniform
// layout with K = the largest rank of the tree (pad_blocks_kernel, into the
// workspace) and the tuned uniform path runs on the padded copies: exact (the
// padded rows and columns are zero), at the cost of one extra pass over the
// generators. Ranks equal within every level need no padding (the per-level
// layout coincides: hss_ranked_run). Plans are cached per thread (last 4).
struct NodeRankPlan {
  RankedPlan Q;               // the per-level plan for K_l
  std::vector<int32_t> K;     // K[l-1], l = 1..p
  bool per_level;             // ranks equal within each level: no padding
  std::vector<hm::PadBlock> blocks;
  int64_t nU, nRW, nB;        // padded sizes (doubles)
  size_t off_U, off_V, off_R, off_W, off_B, off_tab, off_ranked, total;
};

hm_status noderank_plan(const hm_tree* tree, const int32_t* kn, int32_t nrhs, NodeRankPlan* N) {
  hm_status st = check_tree(tree);
  if (st) return st;
  const int p = tree->levels;
  const int64_t n = tree->n, b = tree->leaf;
  if (p > 0 && !kn) return fail(HM_ERR_INVALID_ARG, "node_ranks is NULL");
  auto h = [](int l, int64_t i) { return ((int64_t)1 << l) - 2 + i; };
  N->K.assign(std::max(p, 1), 0);
  N->per_level = true;
  for (int l = 1; l <= p; ++l)
    for (int64_t i = 0; i < ((int64_t)1 << l); ++i) {
      const int k = kn[h(l, i)];
      if (k < 0) return fail(HM_ERR_INVALID_ARG, "node_ranks[%lld] = %d < 0", (long long)h(l, i), k);
      if (k > hm::kMaxRank) return fail(HM_ERR_UNSUPPORTED, "rank %d > %d", k, hm::kMaxRank);
      N->per_level = N->per_level && k == kn[h(l, 0)];
      N->K[l - 1] = std::max(N->K[l - 1], k);
    }
  if (!N->per_level) {
    // pad every level to the largest rank of the tree: the uniform layout, so the
    // tuned uniform kernels run (the per-level ranked kernels are CUDA-core
    // thread-per-output ones: measured 2.2 ms vs ~1.0 ms on a 13-level tree)
    int kmax = 0;
    for (int l = 1; l <= p; ++l) kmax = std::max(kmax, N->K[l - 1]);
    for (int l = 1; l <= p; ++l) N->K[l - 1] = kmax;
  }
  if ((st = hss_ranked_plan(tree, N->K.data(), nrhs, &N->Q))) return st;
  N->blocks.clear();
  N->nU = N->nRW = N->nB = 0;
  size_t off = 0;
  if (!N->per_level && p > 0) {
    const std::vector<int32_t>& K = N->K;
    auto Kl = [&](int l) { return (int64_t)K[l - 1]; };
    N->nU = n * Kl(p);
    for (int l = 1; l < p; ++l) N->nRW += ((int64_t)1 << l) * 2 * Kl(l + 1) * Kl(l);
    for (int l = 1; l <= p; ++l) N->nB += ((int64_t)1 << (l - 1)) * 2 * Kl(l) * Kl(l);
    // one entry per padded block (every padded element written once): compact
    // source offsets walk the arrays in their order, padded ones are per-level
    int64_t su = 0;
    for (int64_t i = 0; i < ((int64_t)1 << p); ++i) {
      const int k = kn[h(p, i)];
      for (int a = 0; a < 2; ++a)
        N->blocks.push_back({su, i * b * Kl(p), (int32_t)b, k, (int32_t)b, (int32_t)Kl(p), a, 0});
      su += b * k;
    }
    int64_t srw = 0, drw = 0;
    for (int l = 1; l < p; ++l) {
      for (int64_t i = 0; i < ((int64_t)1 << l); ++i) {
        const int k = kn[h(l, i)], k0 = kn[h(l + 1, 2 * i)], k1 = kn[h(l + 1, 2 * i + 1)];
        const int64_t dblk = drw + i * 2 * Kl(l + 1) * Kl(l);
        const int32_t dr = (int32_t)Kl(l + 1), dc = (int32_t)Kl(l);
        for (int a = 2; a <= 3; ++a) {
          N->blocks.push_back({srw, dblk, k0, k, dr, dc, a, 0});
          N->blocks.push_back({srw + (int64_t)k0 * k, dblk + Kl(l + 1) * Kl(l), k1, k, dr, dc, a, 0});
        }
        srw += (int64_t)(k0 + k1) * k;
      }
      drw += ((int64_t)1 << l) * 2 * Kl(l + 1) * Kl(l);
    }
    int64_t sb = 0, db = 0;
    for (int l = 1; l <= p; ++l) {
      for (int64_t q = 0; q < ((int64_t)1 << (l - 1)); ++q) {
        const int k0 = kn[h(l, 2 * q)], k1 = kn[h(l, 2 * q + 1)];
        const int64_t dblk = db + q * 2 * Kl(l) * Kl(l);
        const int32_t dk = (int32_t)Kl(l);
        N->blocks.push_back({sb, dblk, k0, k1, dk, dk, 4, 0});
        N->blocks.push_back({sb + (int64_t)k0 * k1, dblk + Kl(l) * Kl(l), k1, k0, dk, dk, 4, 0});
        sb += 2 * (int64_t)k0 * k1;
      }
      db += ((int64_t)1 << (l - 1)) * 2 * Kl(l) * Kl(l);
    }
    N->off_U = off; off = align_up(off + sizeof(double) * (size_t)N->nU);
    N->off_V = off; off = align_up(off + sizeof(double) * (size_t)N->nU);
    N->off_R = off; off = align_up(off + sizeof(double) * (size_t)N->nRW);
    N->off_W = off; off = align_up(off + sizeof(double) * (size_t)N->nRW);
    N->off_B = off; off = align_up(off + sizeof(double) * (size_t)N->nB);
    N->off_tab = off; off = align_up(off + sizeof(hm::PadBlock) * N->blocks.size());
  }
  N->off_ranked = off;
  N->total = off + N->Q.total;
  return HM_OK;
}

hm_status gen_upload_tables(const PinnedImage& img, size_t off_tab, char* w, cudaStream_t s);

// Per-thread cache of the last 4 per-node plans (key: tree, node ranks, nrhs).
struct NodeRankCached {
  int64_t n, leaf;
  int32_t p, nrhs;
  std::vector<int32_t> kn;
  NodeRankPlan N;
  PinnedImage img;
};

const NodeRankCached* noderank_cached(const hm_tree* tree, const int32_t* kn, int32_t nrhs, hm_status* st) {
  thread_local std::vector<NodeRankCached> cache;
  if ((*st = check_tree(tree))) return nullptr;
  const int p = tree->levels;
  const size_t nn = (size_t)((((int64_t)1 << (p + 1)) - 2));
  for (size_t e = 0; e < cache.size(); ++e) {
    const NodeRankCached& c = cache[e];
    if (c.n == tree->n && c.leaf == tree->leaf && c.p == p && c.nrhs == nrhs && kn && c.kn.size() == nn &&
        memcmp(c.kn.data(), kn, nn * sizeof(int32_t)) == 0) {
      if (e) std::rotate(cache.begin(), cache.begin() + e, cache.begin() + e + 1);
      return &cache.front();
    }
  }
  NodeRankCached c;
  c.n = tree->n; c.leaf = tree->leaf; c.p = p; c.nrhs = nrhs;
  if ((*st = noderank_plan(tree, kn, nrhs, &c.N))) return nullptr;
  if (kn) c.kn.assign(kn, kn + nn);
  c.img.host.resize(sizeof(hm::PadBlock) * c.N.blocks.size());
  if (!c.img.empty()) memcpy(c.img.host.data(), c.N.blocks.data(), c.img.size());
  cache.insert(cache.begin(), std::move(c));
  if (cache.size() > 4) cache.pop_back();
  return &cache.front();
}

hm_status hss_noderank_run(const hm_tree* tree, const int32_t* kn, int op, const double* D, const double* U,
                           const double* V, const double* R, const double* W, const double* B, const double* X,
                           int32_t nrhs, double* Y, void* ws, size_t ws_bytes, cudaStream_t s) {
  hm_status st;
  const NodeRankCached* nc = noderank_cached(tree, kn, nrhs, &st);
  if (st) return st;
  const NodeRankPlan& N = nc->N;
  if (!ws || ws_bytes < N.total || !aligned16(ws))
    return fail(HM_ERR_WORKSPACE, "workspace %zu bytes < required %zu (or misaligned)", ws_bytes, N.total);
  char* w = static_cast<char*>(ws);
  if (N.per_level)
    return hss_ranked_run(tree, N.K.data(), op, D, U, V, R, W, B, X, nrhs, Y, w + N.off_ranked,
                          ws_bytes - N.off_ranked, s);
  double* pU = reinterpret_cast<double*>(w + N.off_U);
  double* pV = reinterpret_cast<double*>(w + N.off_V);
  double* pR = reinterpret_cast<double*>(w + N.off_R);
  double* pW = reinterpret_cast<double*>(w + N.off_W);
  double* pB = reinterpret_cast<double*>(w + N.off_B);
  bool needR = false, needB = false, needU = false;
  for (const hm::PadBlock& b : N.blocks) {
    const bool data = b.rows > 0 && b.cols > 0;
    needU = needU || (data && b.arr <= 1);
    needR = needR || (data && (b.arr == 2 || b.arr == 3));
    needB = needB || (data && b.arr == 4);
  }
  if ((needU && (!U || !V)) || (needR && (!R || !W)) || (needB && !B))
    return fail(HM_ERR_INVALID_ARG, "NULL generator pointer");
  g_launches = 0;
  prof_new_call();
  if (!N.blocks.empty()) {
    if ((st = gen_upload_tables(nc->img, N.off_tab, w, s))) return st;
    hm::PadParams pp;
    pp.blocks = reinterpret_cast<const hm::PadBlock*>(w + N.off_tab);
    const double* srcs[5] = {U, V, R, W, B};
    double* dsts[5] = {pU, pV, pR, pW, pB};
    for (int a = 0; a < 5; ++a) {
      pp.src[a] = srcs[a];
      pp.dst[a] = dsts[a];
    }
    if ((st = launch("pad_blocks", s, [&] {
           const int64_t nb = (int64_t)N.blocks.size();
           hm::pad_blocks_kernel<<<(unsigned)std::min<int64_t>(nb, 148 * 8), hm::kThreads, 0, s>>>(pp, nb);
         })))
      return st;
  }
  const int32_t pre = g_launches;
  st = hss_ranked_run(tree, N.K.data(), op, D, pU, pV, pR, pW, pB, X, nrhs, Y, w + N.off_ranked,
                      ws_bytes - N.off_ranked, s);
  g_launches += pre;
  return st;
}

// ---- distributed HSS ----

hm_status hss_dist_plan(const hm_tree* tree, int32_t k, int32_t nrhs, const hm_part* part, int32_t flags,
                        HssPlan* P, DistPart* d) {
  hm_status st = check_tree(tree);
  if (st) return st;
  if ((st = check_part(tree, part, d))) return st;
  return hss_plan_ex(tree->n >> d->q, tree->leaf, tree->levels - d->q, d->q, k, nrhs, flags, P);
}

// ---- distributed HSS: phase bodies ----

hm_status hss_dist_begin_body(const HssPlan& P, const DistPart& d, const double* V_local, const double* W_sub,
                              const double* W_root, const double* X_local, double* send, char* w,
                              cudaStream_t s) {
  if (P.k == 0) return HM_OK;  // block diagonal: nothing to exchange, no tree
  double* xh = reinterpret_cast<double*>(w + P.off_xh);
  if (d.q == 0) {
    // one rank: the whole tree is local and the exchange is empty; Step 1 and
    // the upsweep to level 1 run here (as in hss_matvec), _end does the rest
    if (P.p == 0) return HM_OK;
    if (!X_local || !V_local || (P.p >= 2 && !W_sub)) return fail(HM_ERR_INVALID_ARG, "NULL V / W / X pointer");
    return hss_up_phase(P, V_local, W_sub, X_local, xh, nullptr, nullptr, s);
  }
  if (!X_local || !V_local || !send || (P.p >= 2 && !W_sub) || (P.p >= 1 && !W_root))
    return fail(HM_ERR_INVALID_ARG, "NULL V / W / X / send pointer");
  return hss_up_phase(P, V_local, W_sub, X_local, xh, W_root, send, s);
}

// gathered: the P level-q x blocks in rank order; if it already is the top
// tree's level-q coefficient array (the one-call path), no copy is made.
hm_status hss_dist_end_body(const HssPlan& P, const DistPart& d, const double* D_local, const double* U_local,
                            const double* R_sub, const double* B_sub, const double* R_root, const double* W_top,
                            const double* R_top, const double* B_top, const double* X_local,
                            const double* gathered, double* Y_local, char* w, cudaStream_t s) {
  const int k = P.k;
  if (!D_local || !X_local || !Y_local || !aligned16(D_local))
    return fail(HM_ERR_INVALID_ARG, "NULL or misaligned D / X / Y pointer");
  double* xh = reinterpret_cast<double*>(w + P.off_xh);
  double* yh = reinterpret_cast<double*>(w + P.off_yh);
  double* txh = reinterpret_cast<double*>(w + P.off_txh);
  double* tyh = reinterpret_cast<double*>(w + P.off_tyh);
  unsigned* fl = P.mma_levels ? reinterpret_cast<unsigned*>(w + P.off_flags) : nullptr;
  const int64_t km = (int64_t)k * P.m;
  hm_status st;
  const double* yleaf = nullptr;
  if (k > 0 && d.q == 0 && P.p >= 1) {
    // one rank: coupling + downsweep of the whole (local) tree on the x blocks
    // _begin left in the workspace, then the leaves (as in hss_matvec)
    if (!U_local || !B_sub || (P.p >= 2 && !R_sub)) return fail(HM_ERR_INVALID_ARG, "NULL U / R / B pointer");
    if ((st = hss_tree_phase(P, P.p, nullptr, R_sub, B_sub, xh, yh, nullptr, nullptr, false, true, s, 0, -1, -1, fl)))
      return st;
    yleaf = yh + (((int64_t)1 << P.p) - 2) * km;
  }
  if (k > 0 && d.q > 0) {
    if (!gathered || !U_local || !B_top || (d.q >= 2 && (!W_top || !R_top)) || (P.p >= 1 && (!R_root || !B_sub)) ||
        (P.p >= 2 && !R_sub))
      return fail(HM_ERR_INVALID_ARG, "NULL gathered / generator pointer");
    // replicated top tree: x of level q from the allgather, up q-1..1, down 1..q
    double* tq = txh + (((int64_t)1 << d.q) - 2) * km;
    if (gathered != tq && cudaMemcpyAsync(tq, gathered, sizeof(double) * (size_t)(d.P * km),
                                          cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return cuda_check("copy of the gathered blocks");
    if ((st = hss_tree_phase(P, d.q, W_top, R_top, B_top, txh, tyh, nullptr, nullptr, true, true, s, 0, -1, -1, fl)))
      return st;
    const double* y_root = tyh + (((int64_t)1 << d.q) - 2 + d.rank) * km;
    if (P.p >= 1) {
      // the subtree's x blocks were left in this workspace by _begin
      if ((st = hss_tree_phase(P, P.p, nullptr, R_sub, B_sub, xh, yh, R_root, y_root, false, true, s, 0, -1, -1, fl)))
        return st;
      yleaf = yh + (((int64_t)1 << P.p) - 2) * km;
    } else {
      yleaf = y_root;
    }
  }
  return hss_leaf_phase(P, D_local, U_local, X_local, Y_local, yleaf, s);
}

}  // namespace hmi

using namespace hmi;

extern "C" {

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
  HM_NVTX("hss_norm2_est");
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
  HM_NVTX("hss_matvec");
  return hss_run(tree, k, D, U, V, R, W, B, X, nrhs, Y, workspace, workspace_bytes,
                 static_cast<cudaStream_t>(stream), 0);
}

hm_status hss_matvec_t(const hm_tree* tree, int32_t k, const double* D, const double* U, const double* V,
                       const double* R, const double* W, const double* B, const double* X, int32_t nrhs,
                       double* Y, void* workspace, size_t workspace_bytes, void* stream) {
  HM_NVTX("hss_matvec_t");
  return hss_run(tree, k, D, U, V, R, W, B, X, nrhs, Y, workspace, workspace_bytes,
                 static_cast<cudaStream_t>(stream), 0, 1);
}

hm_status hss_matvec_hostio(const hm_tree* tree, int32_t k, const double* D, const double* U, const double* V,
                            const double* R, const double* W, const double* B, const double* X_host,
                            int32_t nrhs, double* Y_host, void* workspace, size_t workspace_bytes, void* stream) {
  HM_NVTX("hss_matvec_hostio");
  return hss_run(tree, k, D, U, V, R, W, B, X_host, nrhs, Y_host, workspace, workspace_bytes,
                 static_cast<cudaStream_t>(stream), HM_WS_HOSTIO);
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
  HM_NVTX("hss_matvec_dist_begin");
  HssPlan P;
  DistPart d;
  hm_status st = hss_dist_plan(tree, k, nrhs, part, 0, &P, &d);
  if (st) return st;
  if (!workspace || workspace_bytes < P.total || !aligned16(workspace))
    return fail(HM_ERR_WORKSPACE, "workspace too small or misaligned");
  g_launches = 0;
  prof_new_call();
  return hss_dist_begin_body(P, d, V_local, W_sub, W_root, X_local, send, static_cast<char*>(workspace),
                             static_cast<cudaStream_t>(stream));
}

hm_status hss_matvec_dist_end(const hm_tree* tree, int32_t k, const hm_part* part, const double* D_local,
                              const double* U_local, const double* R_sub, const double* B_sub,
                              const double* R_root, const double* W_top, const double* R_top, const double* B_top,
                              const double* X_local, int32_t nrhs, const double* gathered, double* Y_local,
                              void* workspace, size_t workspace_bytes, void* stream) {
  HM_NVTX("hss_matvec_dist_end");
  HssPlan P;
  DistPart d;
  hm_status st = hss_dist_plan(tree, k, nrhs, part, 0, &P, &d);
  if (st) return st;
  if (!workspace || workspace_bytes < P.total || !aligned16(workspace))
    return fail(HM_ERR_WORKSPACE, "workspace too small or misaligned");
  g_launches = 0;
  prof_new_call();
  return hss_dist_end_body(P, d, D_local, U_local, R_sub, B_sub, R_root, W_top, R_top, B_top, X_local, gathered,
                           Y_local, static_cast<char*>(workspace), static_cast<cudaStream_t>(stream));
}

// Per-level ranks.
hm_status hm_hss_ranked_workspace_bytes(const hm_tree* tree, const int32_t* ranks, int32_t nrhs, size_t* bytes) {
  if (!bytes) return fail(HM_ERR_INVALID_ARG, "bytes is NULL");
  RankedPlan Q;
  hm_status st = hss_ranked_plan(tree, ranks, nrhs, &Q);
  if (st) return st;
  *bytes = Q.total;
  return HM_OK;
}

hm_status hss_matvec_ranked(const hm_tree* tree, const int32_t* ranks, int32_t op, const double* D, const double* U,
                            const double* V, const double* R, const double* W, const double* B, const double* X,
                            int32_t nrhs, double* Y, void* workspace, size_t workspace_bytes, void* stream) {
  HM_NVTX("hss_matvec_ranked");
  if (op != 0 && op != 1) return fail(HM_ERR_INVALID_ARG, "op = %d (0: A X, 1: A^T X)", op);
  return hss_ranked_run(tree, ranks, op, D, U, V, R, W, B, X, nrhs, Y, workspace, workspace_bytes,
                        static_cast<cudaStream_t>(stream));
}

// Per-node ranks.
hm_status hm_hss_noderanked_workspace_bytes(const hm_tree* tree, const int32_t* node_ranks, int32_t nrhs,
                                            size_t* bytes) {
  if (!bytes) return fail(HM_ERR_INVALID_ARG, "bytes is NULL");
  hm_status st;
  const NodeRankCached* nc = noderank_cached(tree, node_ranks, nrhs, &st);
  if (st) return st;
  *bytes = nc->N.total;
  return HM_OK;
}

hm_status hss_matvec_noderanked(const hm_tree* tree, const int32_t* node_ranks, int32_t op, const double* D,
                                const double* U, const double* V, const double* R, const double* W, const double* B,
                                const double* X, int32_t nrhs, double* Y, void* workspace, size_t workspace_bytes,
                                void* stream) {
  HM_NVTX("hss_matvec_noderanked");
  if (op != 0 && op != 1) return fail(HM_ERR_INVALID_ARG, "op = %d (0: A X, 1: A^T X)", op);
  return hss_noderank_run(tree, node_ranks, op, D, U, V, R, W, B, X, nrhs, Y, workspace, workspace_bytes,
                          static_cast<cudaStream_t>(stream));
}

// One call, NCCL inside: Step 1 + the subtree upsweep to x of
// node (q, r); the allgather of the P level-q blocks straight into the
// replicated top tree's workspace; the top tree (levels 1..q, every rank
// redundantly), the subtree's coupling + downsweep from y of (q, r), Step 4.
// The exchange is not overlapped: everything after it depends on y of (q, r)
// (DESIGN.md §7 gives the measured cost and why no independent work remains).
hm_status hm_hss_dist_workspace_bytes(const hm_tree* tree, int32_t k, int32_t nrhs, int32_t nranks, size_t* bytes) {
  if (!bytes) return fail(HM_ERR_INVALID_ARG, "bytes is NULL");
  const hm_part part{nranks, 0};
  HssPlan P;
  DistPart d;
  hm_status st = hss_dist_plan(tree, k, nrhs, &part, 0, &P, &d);
  if (st) return st;
  *bytes = P.total;
  return HM_OK;
}

hm_status hss_matvec_dist(hm_comm* comm, const hm_tree* tree, int32_t k, const double* D_local,
                          const double* U_local, const double* V_local, const double* R_sub, const double* W_sub,
                          const double* B_sub, const double* R_root, const double* W_root, const double* R_top,
                          const double* W_top, const double* B_top, const double* X_local, int32_t nrhs,
                          double* Y_local, void* workspace, size_t workspace_bytes, void* stream) {
  HM_NVTX("hss_matvec_dist");
  int32_t nranks = 0, rank = 0;
  hm_status st = comm_check(comm, &nranks, &rank);
  if (st) return st;
  const hm_part part{nranks, rank};
  HssPlan P;
  DistPart d;
  if ((st = hss_dist_plan(tree, k, nrhs, &part, 0, &P, &d))) return st;
  if (!workspace || workspace_bytes < P.total || !aligned16(workspace))
    return fail(HM_ERR_WORKSPACE, "workspace %zu bytes < required %zu (or misaligned)", workspace_bytes, P.total);
  if (X_local && Y_local && overlap(X_local, sizeof(double) * (size_t)(P.n * nrhs), Y_local,
                                    sizeof(double) * (size_t)(P.n * nrhs)))
    return fail(HM_ERR_INVALID_ARG, "X and Y overlap");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(workspace);
  const int64_t km = (int64_t)k * nrhs;
  const int64_t send_doubles = (d.q > 0) ? km : 0;
  // rank r's block goes to its own slot of the level-q coefficient array of
  // the top tree; the allgather then fills every slot in place
  double* tq = reinterpret_cast<double*>(w + P.off_txh) + (((int64_t)1 << d.q) - 2) * km;
  double* send = send_doubles > 0 ? tq + d.rank * km : nullptr;
  g_launches = 0;
  prof_new_call();
  if ((st = hss_dist_begin_body(P, d, V_local, W_sub, W_root, X_local, send, w, s))) return st;
  if ((st = comm_allgather_start(comm, send, send_doubles, tq, s))) return st;
  if ((st = comm_allgather_wait(comm, send_doubles, s))) return st;
  return hss_dist_end_body(P, d, D_local, U_local, R_sub, B_sub, R_root, W_top, R_top, B_top, X_local,
                           send_doubles > 0 ? tq : nullptr, Y_local, w, s);
}

}  // extern "C"
