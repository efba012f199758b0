// hm_convert.cu — hss2hodlr: the exact HODLR
// factors of an HSS matrix from the nested bases of eq. (3).
#include "hm_internal.cuh"
#include "hm_convert.cuh"

using namespace hmi;

extern "C" {

// ------------------------------------------------------ hss2hodlr (f3) --

hm_status hss_to_hodlr(const hm_tree* tree, int32_t k, const double* U, const double* V, const double* R,
                       const double* W, const double* B, double* Uh, double* Vh, void* stream) {
  HM_NVTX("hss_to_hodlr");
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

}  // extern "C"
