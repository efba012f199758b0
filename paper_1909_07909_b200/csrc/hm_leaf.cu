// hm_leaf.cu — launches of the leaf pass: per leaf i,
//   Y(I_i) = D_i X(I_i) + sum_s A_s(I_i) T_s[node_s(i)]
// (HODLR H1 + H3: Fig. 5 left's "if A is dense return Av" plus every level's
// U_l t_l; HSS Step 4: U_i y_i + D_i X(I_i)). The
// kernels are in hm_fast.cuh (tuned) and hm_kernels.cuh (generic).
#include "hm_internal.cuh"

namespace hmi {
namespace {

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
  const unsigned grid = (unsigned)std::min<int64_t>(nleaves, num_sms());
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

template <int RG, int NT, int KT>
hm_status launch_leaf_down(const hm::LeafParams& lp, const hm::LeafDownParams& q, int64_t nleaves, cudaStream_t s) {
  constexpr int PF = LeafMmaTune<RG, NT>::PF, MINB = LeafMmaTune<RG, NT>::MINB;
  const size_t smem = sizeof(double) * (size_t)((lp.b + 2 * KT) * (NT * 8 + 2));
  if (smem > sizeof(double) * (size_t)kSmemBudgetDoubles) return HM_ERR_UNSUPPORTED;
  const int64_t chunks = (lp.m + NT * 8 - 1) / (NT * 8);
  allow_smem(hm::leaf_mma_down_kernel<RG, NT, PF, MINB, KT>, smem);
  return launch("leaf_mma_down", s, [&] {
    hm::leaf_mma_down_kernel<RG, NT, PF, MINB, KT><<<(unsigned)(nleaves * chunks), 256, smem, s>>>(lp, q);
  });
}

}  // namespace

bool leaf_down_supported(int64_t b, int k, int nt) {
  const int rg = (int)(b / 64);
  const bool inst = b % 64 == 0 && (k == 16 || k == 32) && (rg == 1 || rg == 2 || rg == 4) &&
                    (nt == 1 || nt == 2 || (nt == 4 && rg < 4));
  return inst && (b + 2 * k) * (nt * 8 + 2) <= kSmemBudgetDoubles;
}

hm_status leaf_down_dispatch(const hm::LeafParams& lp, const hm::LeafDownParams& q, int64_t nleaves, int k, int nt,
                             cudaStream_t s) {
  if (lp.nseg != 1 || lp.dtrans || q.p < 2 || !leaf_down_supported(lp.b, k, nt)) return HM_ERR_UNSUPPORTED;
  const int rg = (int)(lp.b / 64);
  if (lp.b % 64 != 0) return HM_ERR_UNSUPPORTED;
#define HM_LD(RG_, NT_)                                                                      \
  if (rg == RG_ && nt == NT_)                                                                \
    return k == 16 ? launch_leaf_down<RG_, NT_, 16>(lp, q, nleaves, s) : launch_leaf_down<RG_, NT_, 32>(lp, q, nleaves, s);
  HM_LD(1, 1) HM_LD(1, 2) HM_LD(1, 4) HM_LD(2, 1) HM_LD(2, 2) HM_LD(2, 4) HM_LD(4, 1) HM_LD(4, 2)
#undef HM_LD
  return HM_ERR_UNSUPPORTED;
}

hm_status leaf_dispatch(const hm::LeafParams& lp, int64_t nleaves, LeafPath path, int k, int nt, int mc,
                        cudaStream_t s, bool kvary) {
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
}  // namespace hmi
