// hm_vt.cu — launches of the right contractions t = V^T X: HODLR H2
// (t_{l,j} = V_l(I_j)^T X(I_j) for every level in one pass) and
// HSS Step 1 (x_i = V_i^T X(I_i)) / the single-block products of the
// distributed top tree. Kernels: hm_fast.cuh (tuned), hm_kernels.cuh (generic).
#include "hm_internal.cuh"

namespace hmi {

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
    hm::vt_lv_kernel<KT, NT, IPW, HM_VT_LV_R, NS, NW><<<(unsigned)(vp.n / vp.tile), NW * 32, smem, s>>>(vp, b);
  });
}

hm_status vt_lv_dispatch(const hm::VtParams& vp, int64_t b, int k, cudaStream_t s) {
  constexpr int R = HM_VT_LV_R, NW = HM_VT_LV_NW, MC = 8 * HM_VT_LV_NT;
  if (HM_VT_LV_MIN_M <= 0 || vp.m < HM_VT_LV_MIN_M || !(k == 16 || k == 32) || b % R != 0 || vp.nlev < 1 ||
      !(vp.tile == 8 * b || vp.tile == 4 * b))
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
}  // namespace hmi
