/*
 * fill.c — fast host fill of the closed-form inverse-Laplacian generators
 * (BASELINE.json config 5; reading G11) for hm_inputs. INPUT
 * GENERATION ONLY: the same bits as hm_inputs' numpy / torch fills (an exact
 * integer product, then one correctly rounded IEEE division), written with
 * OpenMP so a 34 GB leaf array takes seconds instead of minutes. Serves both
 * sides (oracle and CUDA path) like the rest of hm_inputs; holds none of the
 * method's arithmetic.
 */
#include <stdint.h>

/* D_i = A(I_i, I_i), A_ij = min(i,j)(n+1-max(i,j))/(n+1) (1-based), for the
 * leaves leaf0 .. leaf0 + nleaves - 1 of the uniform tree with leaf size b. */
int fill_laplacian_leaves(int64_t n, int64_t b, int64_t leaf0, int64_t nleaves, double* out) {
  if (n < 1 || b < 1 || leaf0 < 0 || nleaves < 0 || (leaf0 + nleaves) * b > n || !out) return -1;
  const double np1 = (double)(n + 1);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < nleaves; ++t) {
    const int64_t base = (leaf0 + t) * b; /* 0-based first row */
    double* blk = out + t * b * b;
    for (int64_t r = 0; r < b; ++r) {
      const int64_t i = base + r + 1;
      for (int64_t c = 0; c < b; ++c) {
        const int64_t j = base + c + 1;
        const int64_t mn = i < j ? i : j, mx = i < j ? j : i;
        blk[r * b + c] = (double)(mn * (n + 1 - mx)) / np1;
      }
    }
  }
  return 0;
}
