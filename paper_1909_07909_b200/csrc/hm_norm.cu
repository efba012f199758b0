// hm_norm.cu — ||A||_2 estimate by the power method on A A^* (SURVEY §8(f)
// f2; "estimating ||A||_2 by means of the power method on AA^*"):
// libhm's own products plus fixed-order vector reductions (hm_vec.cuh).
#include "hm_internal.cuh"
#include "hm_vec.cuh"

namespace hmi {

// ------------------------------------------------ norm estimate (f2) --
//
// Power method on A A^* (SURVEY §8(f) f2), nrhs = 1:
//   v = x0/||x0||; iters times: w = A^T v, eta = ||w|| (-> est), z = A w, v = z/||z||.
// Workspace: [matvec workspace][v: n][w: n][norm partials]; every product is
// libhm's own matvec / adjoint on the same workspace.
NormPlan norm_plan(size_t mv_bytes, int64_t n) {
  NormPlan N;
  size_t off = align_up(mv_bytes);
  N.off_v = off; off = align_up(off + sizeof(double) * (size_t)n);
  N.off_w = off; off = align_up(off + sizeof(double) * (size_t)n);
  N.off_part = off; off = align_up(off + sizeof(double) * hm::kVecMaxBlocks);
  N.total = off;
  return N;
}

hm_status power_norm2(int64_t n, const double* x0, int32_t iters, double* est, char* w, const NormPlan& N,
                      cudaStream_t s, const std::function<hm_status(int, const double*, double*)>& apply) {
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

}  // namespace hmi
