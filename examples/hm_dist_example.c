/*
 * hm_dist_example.c — the distributed product from plain C (no Python, no
 * torch): P processes, one per GPU (rank r on device r), each owning the rows
 * of the level-q node (q, r) of the cluster tree (P = 2^q; include/hm.h
 * "multi-GPU"). Rank 0 creates the communicator id and hands it to the other
 * ranks through pipes; every rank then calls hodlr_matvec_dist and
 * hss_matvec_dist once on its local generators of the inverse 1D Laplacian
 * (HODLR rank 1 per level, G11; HSS rank 2, R = W = [I; I], constant
 * cores) and checks its rows of Y against the O(n) closed form
 *   y_i = [(n+1-i) sum_{j<=i} j x_j + i sum_{j>i} (n+1-j) x_j] / (n+1).
 *
 *   hm_dist_example [P]          P processes (default 1), P GPUs
 *   hm_dist_example --host-only  workspace queries + a communicator id (no GPU)
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/wait.h>
#include <unistd.h>

#include "hm.h"

typedef int cudaError_t;
extern cudaError_t cudaMalloc(void** p, size_t n);
extern cudaError_t cudaFree(void* p);
extern cudaError_t cudaMemcpy(void* d, const void* s, size_t n, int kind);
extern cudaError_t cudaDeviceSynchronize(void);
extern cudaError_t cudaSetDevice(int dev);

enum { H2D = 1, D2H = 2 };

static void* dev_copy(const double* h, size_t count) {
  void* d = NULL;
  if (cudaMalloc(&d, sizeof(double) * (count ? count : 1)) != 0) return NULL;
  if (count) cudaMemcpy(d, h, sizeof(double) * count, H2D);
  return d;
}

static double x_of(int64_t i) { return sin(0.37 * (double)i) + 0.1; } /* 0-based row */

/* inverse-Laplacian entry, 1-based (i, j) */
static double lap(int64_t n, int64_t i, int64_t j) {
  const int64_t mn = i < j ? i : j, mx = i < j ? j : i;
  return (double)(mn * (n + 1 - mx)) / (double)(n + 1);
}

static int run_rank(int P, int rank, const unsigned char* id) {
  const int32_t p = 8;
  const int64_t b = 64, n = b << p, nl = n / P;
  int q = 0;
  while ((1 << q) < P) ++q;
  if (cudaSetDevice(rank) != 0) {
    fprintf(stderr, "rank %d: no device %d\n", rank, rank);
    return 1;
  }
  hm_comm* comm = NULL;
  if (hm_comm_init(P, rank, id, &comm) != HM_OK) {
    fprintf(stderr, "rank %d: hm_comm_init: %s\n", rank, hm_last_error());
    return 1;
  }
  hm_tree tree = {n, p, 0, b};
  const int64_t r0 = (int64_t)rank * nl; /* first global row (0-based) */
  const int64_t lpr = ((int64_t)1 << p) / P;
  /* closed-form Y for the local rows */
  double* yref = malloc(sizeof(double) * nl);
  {
    double s_lo = 0, s_hi = 0; /* sum_{j<=i} j x_j, sum_{j>i} (n+1-j) x_j (1-based) */
    for (int64_t j = 1; j <= n; ++j) s_hi += (double)(n + 1 - j) * x_of(j - 1);
    for (int64_t i = 1; i <= n; ++i) {
      s_lo += (double)i * x_of(i - 1);
      s_hi -= (double)(n + 1 - i) * x_of(i - 1);
      if (i - 1 >= r0 && i - 1 < r0 + nl)
        yref[i - 1 - r0] = ((double)(n + 1 - i) * s_lo + (double)i * s_hi) / (double)(n + 1);
    }
  }
  double* X = malloc(sizeof(double) * nl);
  double* Y = malloc(sizeof(double) * nl);
  for (int64_t r = 0; r < nl; ++r) X[r] = x_of(r0 + r);
  double* D = malloc(sizeof(double) * nl * b);
  for (int64_t L = 0; L < lpr; ++L)
    for (int64_t r = 0; r < b; ++r)
      for (int64_t c = 0; c < b; ++c) {
        const int64_t g = (rank * lpr + L) * b; /* first global row of the leaf */
        D[(L * b + r) * b + c] = lap(n, g + r + 1, g + c + 1);
      }
  int rc = 0;
  void *dD = dev_copy(D, nl * b), *dX = dev_copy(X, nl), *dY = dev_copy(NULL, nl);

  /* ---- HODLR: U_l, V_l rows I_r of every level (rank 1 each, G11) */
  {
    int32_t ranks[8];
    for (int l = 0; l < p; ++l) ranks[l] = 1;
    double* U = malloc(sizeof(double) * nl * p);
    double* V = malloc(sizeof(double) * nl * p);
    for (int32_t l = 1; l <= p; ++l)
      for (int64_t r = 0; r < nl; ++r) {
        const int64_t i = r0 + r + 1, a = (r0 + r) / (n >> l);
        U[(l - 1) * nl + r] = (a & 1) ? (double)(n + 1 - i) : (double)i;
        V[(l - 1) * nl + r] = (a & 1) ? (double)(n + 1 - i) / (double)(n + 1) : (double)i / (double)(n + 1);
      }
    size_t ws = 0;
    void *dU = dev_copy(U, nl * p), *dV = dev_copy(V, nl * p), *dW = NULL;
    if (hm_hodlr_dist_workspace_bytes(&tree, ranks, 1, P, &ws) != HM_OK || cudaMalloc(&dW, ws) != 0) rc = 1;
    if (!rc && hodlr_matvec_dist(comm, &tree, ranks, dD, dU, dV, dX, 1, dY, dW, ws, NULL) != HM_OK) {
      fprintf(stderr, "rank %d: hodlr_matvec_dist: %s\n", rank, hm_last_error());
      rc = 1;
    }
    cudaDeviceSynchronize();
    cudaMemcpy(Y, dY, sizeof(double) * nl, D2H);
    double e = 0, nr = 0;
    for (int64_t r = 0; r < nl; ++r) {
      e += (Y[r] - yref[r]) * (Y[r] - yref[r]);
      nr += yref[r] * yref[r];
    }
    printf("rank %d/%d: hodlr_matvec_dist rows %lld..%lld relerr %.3e\n", rank, P, (long long)r0,
           (long long)(r0 + nl), sqrt(e / nr));
    if (!(sqrt(e / nr) <= 1e-12)) rc = 1;
    cudaFree(dU); cudaFree(dV); cudaFree(dW);
    free(U); free(V);
  }

  /* ---- HSS: exact rank-2 form, U = [i, n+1-i], V = U / (n+1), R = W = [I2; I2],
   * B12 = [[0,1],[0,0]], B21 = [[0,0],[1,0]] on every node: the shards are copies */
  {
    const int32_t k = 2, pl = p - q;
    double* U = malloc(sizeof(double) * nl * 2);
    double* V = malloc(sizeof(double) * nl * 2);
    for (int64_t r = 0; r < nl; ++r) {
      const double i = (double)(r0 + r + 1);
      U[2 * r] = i;
      U[2 * r + 1] = (double)(n + 1) - i;
      V[2 * r] = U[2 * r] / (double)(n + 1);
      V[2 * r + 1] = U[2 * r + 1] / (double)(n + 1);
    }
    const double Rn[8] = {1, 0, 0, 1, 1, 0, 0, 1};
    const double Bn[8] = {0, 1, 0, 0, 0, 0, 1, 0};
    const int64_t nsub_t = ((int64_t)1 << pl) - 2, nsub_b = ((int64_t)1 << pl) - 1;
    const int64_t ntop_t = q >= 2 ? ((int64_t)1 << q) - 2 : 0, ntop_b = q >= 1 ? ((int64_t)1 << q) - 1 : 0;
    int64_t cnt = nsub_t > ntop_t ? nsub_t : ntop_t;
    if (nsub_b > cnt) cnt = nsub_b;
    if (cnt < 1) cnt = 1;
    double* Rs = malloc(sizeof(double) * 8 * cnt);
    double* Bs = malloc(sizeof(double) * 8 * cnt);
    for (int64_t t = 0; t < cnt; ++t) {
      memcpy(Rs + 8 * t, Rn, sizeof Rn);
      memcpy(Bs + 8 * t, Bn, sizeof Bn);
    }
    void *dU = dev_copy(U, nl * 2), *dV = dev_copy(V, nl * 2);
    void *dR = dev_copy(Rs, 8 * cnt), *dB = dev_copy(Bs, 8 * cnt), *dW = NULL;
    size_t ws = 0;
    if (hm_hss_dist_workspace_bytes(&tree, k, 1, P, &ws) != HM_OK || cudaMalloc(&dW, ws) != 0) rc = 1;
    /* R_sub = W_sub, B_sub, R_root = W_root (q >= 1), R_top = W_top, B_top: all copies */
    if (!rc && hss_matvec_dist(comm, &tree, k, dD, dU, dV, dR, dR, dB, q >= 1 ? dR : NULL, q >= 1 ? dR : NULL,
                               ntop_t ? dR : NULL, ntop_t ? dR : NULL, ntop_b ? dB : NULL, dX, 1, dY, dW, ws,
                               NULL) != HM_OK) {
      fprintf(stderr, "rank %d: hss_matvec_dist: %s\n", rank, hm_last_error());
      rc = 1;
    }
    cudaDeviceSynchronize();
    cudaMemcpy(Y, dY, sizeof(double) * nl, D2H);
    double e = 0, nr = 0;
    for (int64_t r = 0; r < nl; ++r) {
      e += (Y[r] - yref[r]) * (Y[r] - yref[r]);
      nr += yref[r] * yref[r];
    }
    printf("rank %d/%d: hss_matvec_dist relerr %.3e\n", rank, P, sqrt(e / nr));
    if (!(sqrt(e / nr) <= 1e-12)) rc = 1;
    cudaFree(dU); cudaFree(dV); cudaFree(dR); cudaFree(dB); cudaFree(dW);
    free(U); free(V); free(Rs); free(Bs);
  }
  if (hm_comm_destroy(comm) != HM_OK) rc = 1;
  cudaFree(dD); cudaFree(dX); cudaFree(dY);
  free(D); free(X); free(Y); free(yref);
  return rc;
}

int main(int argc, char** argv) {
  if (argc > 1 && strcmp(argv[1], "--host-only") == 0) {
    hm_tree tree = {64 << 8, 8, 0, 64};
    int32_t ranks[8] = {1, 1, 1, 1, 1, 1, 1, 1};
    size_t w1 = 0, w2 = 0;
    unsigned char id[HM_COMM_ID_BYTES];
    if (hm_hodlr_dist_workspace_bytes(&tree, ranks, 1, 4, &w1) != HM_OK ||
        hm_hss_dist_workspace_bytes(&tree, 2, 1, 4, &w2) != HM_OK || hm_comm_unique_id(id) != HM_OK) {
      fprintf(stderr, "host-only: %s\n", hm_last_error());
      return 1;
    }
    if (hm_hodlr_dist_workspace_bytes(&tree, ranks, 1, 3, &w1) != HM_ERR_UNSUPPORTED) return 1;
    printf("host-only: workspaces %zu / %zu bytes at P = 4, communicator id created, P = 3 rejected\n", w1, w2);
    return 0;
  }
  const int P = argc > 1 ? atoi(argv[1]) : 1;
  if (P < 1 || (P & (P - 1))) {
    fprintf(stderr, "P must be a power of two\n");
    return 2;
  }
  int fds[64][2];
  for (int r = 1; r < P; ++r)
    if (pipe(fds[r]) != 0) return 2;
  int rank = 0;
  for (int r = 1; r < P; ++r) {
    const pid_t pid = fork(); /* before any CUDA / NCCL call */
    if (pid == 0) {
      rank = r;
      break;
    }
  }
  unsigned char id[HM_COMM_ID_BYTES];
  if (rank == 0) {
    if (hm_comm_unique_id(id) != HM_OK) {
      fprintf(stderr, "hm_comm_unique_id: %s\n", hm_last_error());
      return 1;
    }
    for (int r = 1; r < P; ++r)
      if (write(fds[r][1], id, sizeof id) != (ssize_t)sizeof id) return 1;
  } else if (read(fds[rank][0], id, sizeof id) != (ssize_t)sizeof id) {
    return 1;
  }
  int rc = run_rank(P, rank, id);
  if (rank == 0) {
    for (int r = 1; r < P; ++r) {
      int status = 0;
      wait(&status);
      if (!WIFEXITED(status) || WEXITSTATUS(status) != 0) rc = 1;
    }
    printf("%s\n", rc ? "FAILED" : "all ranks OK");
  }
  return rc;
}
