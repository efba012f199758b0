/*
 * hm_matvec_example.c — calling libhm from plain C (no Python, no torch):
 * Y = A X for the HODLR matrix of the inverse 1D Laplacian (BASELINE.json
 * config 5 structure, scaled down), checked with tridiag(-1,2,-1) Y = X.
 *
 *   cc -I include examples/hm_matvec_example.c -L paper_1909_07909_b200 -lhm_link \
 *      -lcudart ... (see tests/test_abi.py::test_c_example_links_and_validates)
 *
 * Without a GPU the program exercises the host side only: it queries the
 * workspace, and a call with an invalid tree must fail on the host with
 * HM_ERR_UNSUPPORTED and a message (argument `--host-only`).
 * With a GPU it allocates device memory with the CUDA runtime, fills the
 * generators from the closed form (G11 of DESIGN.md), runs hodlr_matvec and
 * hodlr_matvec_t and prints the tridiagonal residual.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "hm.h"

/* minimal CUDA runtime declarations (the example links libcudart dynamically
 * only when run with a GPU; the host-only path needs none of them) */
typedef int cudaError_t;
extern cudaError_t cudaMalloc(void** p, size_t n);
extern cudaError_t cudaFree(void* p);
extern cudaError_t cudaMemcpy(void* d, const void* s, size_t n, int kind);
extern cudaError_t cudaDeviceSynchronize(void);
extern cudaError_t cudaGetDeviceCount(int* n);

int main(int argc, char** argv) {
  const int host_only = argc > 1 && strcmp(argv[1], "--host-only") == 0;
  const int32_t p = 6;
  const int64_t b = 64, n = b << p;
  hm_tree tree = {n, p, 0, b};
  int32_t ranks[6] = {1, 1, 1, 1, 1, 1};
  size_t ws = 0;
  if (hm_hodlr_workspace_bytes(&tree, ranks, 1, 0, &ws) != HM_OK) {
    fprintf(stderr, "workspace query failed: %s\n", hm_last_error());
    return 1;
  }
  hm_tree bad = {n + 1, p, 0, b};
  if (hodlr_matvec(&bad, ranks, NULL, NULL, NULL, NULL, 1, NULL, NULL, 0, NULL) != HM_ERR_UNSUPPORTED ||
      strlen(hm_last_error()) == 0) {
    fprintf(stderr, "invalid tree not rejected on the host\n");
    return 1;
  }
  printf("abi %d, workspace %zu bytes, invalid tree rejected: %s\n", hm_abi_version(), ws, hm_last_error());
  if (host_only) return 0;

  /* closed-form generators (1-based i, j): D from min(i,j)(n+1-max(i,j))/(n+1);
   * level l rows of node a: upper block (a even) u = i, v = (n+1-j)/(n+1);
   * lower block (a odd) u = n+1-i, v = j/(n+1) — DESIGN.md G11 */
  double* D = malloc(sizeof(double) * n * b);
  double* U = malloc(sizeof(double) * n * p);
  double* V = malloc(sizeof(double) * n * p);
  double* X = malloc(sizeof(double) * n);
  double* Y = malloc(sizeof(double) * n);
  const double np1 = (double)(n + 1);
  for (int64_t L = 0; L < (1 << p); ++L)
    for (int64_t r = 0; r < b; ++r)
      for (int64_t c = 0; c < b; ++c) {
        const int64_t i = L * b + r + 1, j = L * b + c + 1;
        const int64_t mn = i < j ? i : j, mx = i < j ? j : i;
        D[(L * b + r) * b + c] = (double)(mn * (n + 1 - mx)) / np1;
      }
  for (int32_t l = 1; l <= p; ++l)
    for (int64_t r = 0; r < n; ++r) {
      const int64_t i = r + 1, a = r / (n >> l);
      U[(l - 1) * n + r] = (a & 1) ? (double)(n + 1 - i) : (double)i;
      V[(l - 1) * n + r] = (a & 1) ? (double)(n + 1 - i) / np1 : (double)i / np1;
    }
  for (int64_t r = 0; r < n; ++r) X[r] = sin(0.37 * (double)r) + 0.1;
  void *dD, *dU, *dV, *dX, *dY, *dW;
  cudaMalloc(&dD, sizeof(double) * n * b);
  cudaMalloc(&dU, sizeof(double) * n * p);
  cudaMalloc(&dV, sizeof(double) * n * p);
  cudaMalloc(&dX, sizeof(double) * n);
  cudaMalloc(&dY, sizeof(double) * n);
  cudaMalloc(&dW, ws);
  cudaMemcpy(dD, D, sizeof(double) * n * b, 1);
  cudaMemcpy(dU, U, sizeof(double) * n * p, 1);
  cudaMemcpy(dV, V, sizeof(double) * n * p, 1);
  cudaMemcpy(dX, X, sizeof(double) * n, 1);
  for (int op = 0; op < 2; ++op) {
    hm_status st = (op ? hodlr_matvec_t : hodlr_matvec)(&tree, ranks, dD, dU, dV, dX, 1, dY, dW, ws, NULL);
    if (st != HM_OK) {
      fprintf(stderr, "matvec failed: %s\n", hm_last_error());
      return 1;
    }
    cudaDeviceSynchronize();
    cudaMemcpy(Y, dY, sizeof(double) * n, 2);
    double num = 0, ny = 0, nx = 0;
    for (int64_t r = 0; r < n; ++r) {
      const double ty = 2 * Y[r] - (r > 0 ? Y[r - 1] : 0) - (r + 1 < n ? Y[r + 1] : 0);
      num += (ty - X[r]) * (ty - X[r]);
      ny += Y[r] * Y[r];
      nx += X[r] * X[r];
    }
    const double res = sqrt(num) / (4 * sqrt(ny) + sqrt(nx));
    printf("%s: tridiag residual %.3e\n", op ? "A^T X" : "A X", res);
    if (!(res < 1e-14)) return 1;
  }
  cudaFree(dD); cudaFree(dU); cudaFree(dV); cudaFree(dX); cudaFree(dY); cudaFree(dW);
  free(D); free(U); free(V); free(X); free(Y);
  return 0;
}
