/*
 * oracle_sanitize_main.c — drives every entry point of oracle/hm_oracle.c on
 * small trees with the awkward shapes (empty and ragged leaves, rank-0 levels
 * and nodes, depth 0 and 1, one right-hand side and several), built with
 * -fsanitize=address,undefined (tests/test_oracle_sanitize.py). Every
 * structured product is also checked against the dense matrix the oracle
 * builds from the same generators (Def. 2.2, eq. (3)), so
 * an out-of-bounds index that happens to read plausible memory still fails.
 * Exit status 0 = clean; the sanitizers abort on the first finding.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "hm_oracle.h"

static uint64_t g_state = 0x9e3779b97f4a7c15ull;
static double urand(void) { /* xorshift64*, uniform in [-1, 1) */
  g_state ^= g_state >> 12;
  g_state ^= g_state << 25;
  g_state ^= g_state >> 27;
  return (double)((g_state * 2685821657736338717ull) >> 11) / 4503599627370496.0 - 1.0;
}
static double* rnd(int64_t count) {
  double* a = (double*)malloc(sizeof(double) * (size_t)(count > 0 ? count : 1));
  for (int64_t i = 0; i < count; ++i) a[i] = urand();
  return a;
}
static int g_fail = 0;
static void check(const char* what, const double* y, const double* ref, int64_t count) {
  double num = 0, den = 0;
  for (int64_t i = 0; i < count; ++i) {
    num += (y[i] - ref[i]) * (y[i] - ref[i]);
    den += ref[i] * ref[i];
  }
  const double rel = den > 0 ? sqrt(num / den) : sqrt(num);
  if (!(rel <= 1e-12)) {
    fprintf(stderr, "MISMATCH %s: relerr %.3e\n", what, rel);
    g_fail = 1;
  }
}
static void must(int rc, const char* what) {
  if (rc != 0) {
    fprintf(stderr, "FAILED %s: rc %d\n", what, rc);
    g_fail = 1;
  }
}
static int64_t leaf_rows(const int64_t* c, int64_t i) { return c[i] - (i ? c[i - 1] : 0); }
static int64_t dblocks(const int64_t* c, int32_t p) {
  int64_t s = 0;
  for (int64_t i = 0; i < (1ll << p); ++i) s += leaf_rows(c, i) * leaf_rows(c, i);
  return s;
}
static void dense_apply(int64_t n, const double* A, const double* X, int32_t m, double* Y, int trans) {
  if (!trans) {
    must(oracle_dense_matvec(n, A, X, m, Y), "dense");
    return;
  }
  double* At = (double*)malloc(sizeof(double) * (size_t)(n * n > 0 ? n * n : 1));
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) At[j * n + i] = A[i * n + j];
  must(oracle_dense_matvec(n, At, X, m, Y), "dense^T");
  free(At);
}
/* Dsel: the diagonal blocks of the listed leaves, in list order */
static double* dsel(const double* D, const int64_t* c, int32_t p, const int64_t* leaves, int64_t nl, int64_t* rows) {
  int64_t tot = 0, rr = 0;
  for (int64_t t = 0; t < nl; ++t) tot += leaf_rows(c, leaves[t]) * leaf_rows(c, leaves[t]);
  double* out = (double*)malloc(sizeof(double) * (size_t)(tot > 0 ? tot : 1));
  int64_t o = 0;
  for (int64_t t = 0; t < nl; ++t) {
    int64_t off = 0;
    for (int64_t i = 0; i < leaves[t]; ++i) off += leaf_rows(c, i) * leaf_rows(c, i);
    const int64_t s = leaf_rows(c, leaves[t]) * leaf_rows(c, leaves[t]);
    memcpy(out + o, D + off, sizeof(double) * (size_t)s);
    o += s;
    rr += leaf_rows(c, leaves[t]);
  }
  (void)p;
  *rows = rr;
  return out;
}
static void gather_rows(const double* Y, const int64_t* c, const int64_t* leaves, int64_t nl, int32_t m, double* out) {
  int64_t o = 0;
  for (int64_t t = 0; t < nl; ++t) {
    const int64_t r0 = leaves[t] ? c[leaves[t] - 1] : 0, r = leaf_rows(c, leaves[t]);
    memcpy(out + o * m, Y + r0 * m, sizeof(double) * (size_t)(r * m));
    o += r;
  }
}

static void hodlr_case(const char* name, int64_t n, int32_t p, const int64_t* c, const int32_t* ranks, int32_t m) {
  int64_t ksum = 0;
  for (int l = 0; l < p; ++l) ksum += ranks[l];
  double *D = rnd(dblocks(c, p)), *U = rnd(n * ksum), *V = rnd(n * ksum), *X = rnd(n * m);
  double *Y = rnd(n * m), *R = rnd(n * m), *A = rnd(n * n);
  must(oracle_hodlr_dense(n, p, c, ranks, D, U, V, A), name);
  for (int trans = 0; trans < 2; ++trans) {
    must((trans ? oracle_hodlr_matvec_t : oracle_hodlr_matvec)(n, p, c, ranks, D, U, V, X, m, Y), name);
    dense_apply(n, A, X, m, R, trans);
    check(name, Y, R, n * m);
    const int64_t leaves[3] = {0, (1ll << p) - 1, (1ll << p) / 2};
    const int64_t nl = p ? 3 : 1;
    int64_t rows = 0;
    double* Ds = dsel(D, c, p, leaves, nl, &rows);
    double *Yl = rnd(rows * m), *Rl = rnd(rows * m);
    must((trans ? oracle_hodlr_matvec_t_leaves : oracle_hodlr_matvec_leaves)(n, p, c, ranks, Ds, U, V, X, m, leaves,
                                                                             nl, Yl),
         name);
    gather_rows(R, c, leaves, nl, m, Rl);
    check(name, Yl, Rl, rows * m);
    free(Ds); free(Yl); free(Rl);
  }
  double est = 0;
  must(oracle_hodlr_norm2_est(n, p, c, ranks, D, U, V, X, 3, &est), name);
  free(D); free(U); free(V); free(X); free(Y); free(R); free(A);
}

static void hss_case(const char* name, int64_t n, int32_t p, const int64_t* c, int32_t k, int32_t m) {
  const int64_t nodes = (1ll << p) - 2 > 0 ? (1ll << p) - 2 : 0;
  double *D = rnd(dblocks(c, p)), *U = rnd(n * k), *V = rnd(n * k), *Rt = rnd(nodes * 2 * k * k),
         *W = rnd(nodes * 2 * k * k), *B = rnd(((1ll << p) - 1) * 2 * k * k), *X = rnd(n * m);
  double *Y = rnd(n * m), *R = rnd(n * m), *A = rnd(n * n);
  must(oracle_hss_dense(n, p, c, k, D, U, V, Rt, W, B, A), name);
  for (int trans = 0; trans < 2; ++trans) {
    must((trans ? oracle_hss_matvec_t : oracle_hss_matvec)(n, p, c, k, D, U, V, Rt, W, B, X, m, Y), name);
    dense_apply(n, A, X, m, R, trans);
    check(name, Y, R, n * m);
    const int64_t leaves[3] = {(1ll << p) - 1, 0, (1ll << p) / 2};
    const int64_t nl = p ? 3 : 1;
    int64_t rows = 0;
    double* Ds = dsel(D, c, p, leaves, nl, &rows);
    double *Yl = rnd(rows * m), *Rl = rnd(rows * m);
    must((trans ? oracle_hss_matvec_t_leaves : oracle_hss_matvec_leaves)(n, p, c, k, Ds, U, V, Rt, W, B, X, m, leaves,
                                                                         nl, Yl),
         name);
    gather_rows(R, c, leaves, nl, m, Rl);
    check(name, Yl, Rl, rows * m);
    free(Ds); free(Yl); free(Rl);
  }
  /* hss2hodlr: the HODLR matrix of the converted factors equals the HSS matrix */
  if (p >= 1) {
    double *Uh = rnd((int64_t)p * n * k), *Vh = rnd((int64_t)p * n * k), *Ah = rnd(n * n);
    int32_t rk[32];
    for (int l = 0; l < p; ++l) rk[l] = k;
    must(oracle_hss_to_hodlr(n, p, c, k, U, V, Rt, W, B, Uh, Vh), name);
    must(oracle_hodlr_dense(n, p, c, rk, D, Uh, Vh, Ah), name);
    check(name, Ah, A, n * n);
    free(Uh); free(Vh); free(Ah);
  }
  /* the same generators through the per-level and per-node layouts */
  if (p >= 1) {
    int32_t rk[32];
    for (int l = 0; l < p; ++l) rk[l] = k;
    must(oracle_hss_matvec_ranked(n, p, c, rk, D, U, V, Rt, W, B, X, m, Y), name);
    dense_apply(n, A, X, m, R, 0);
    check(name, Y, R, n * m);
  }
  double est = 0;
  must(oracle_hss_norm2_est(n, p, c, k, D, U, V, Rt, W, B, X, 3, &est), name);
  free(D); free(U); free(V); free(Rt); free(W); free(B); free(X); free(Y); free(R); free(A);
}

static void hss_ranked_case(const char* name, int64_t n, int32_t p, const int64_t* c, const int32_t* ranks, int32_t m) {
  /* sizes from the layout in hm_oracle.h (k_l = ranks[l-1]) */
  const int64_t kp = ranks[p - 1];
  int64_t rw = 0, bb = 0;
  for (int l = 1; l < p; ++l) rw += (1ll << l) * 2 * ranks[l] * ranks[l - 1];
  for (int l = 1; l <= p; ++l) bb += (1ll << (l - 1)) * 2 * ranks[l - 1] * ranks[l - 1];
  double *D = rnd(dblocks(c, p)), *U = rnd(n * kp), *V = rnd(n * kp), *Rt = rnd(rw), *W = rnd(rw), *B = rnd(bb),
         *X = rnd(n * m), *Y = rnd(n * m), *R = rnd(n * m), *A = rnd(n * n);
  must(oracle_hss_dense_ranked(n, p, c, ranks, D, U, V, Rt, W, B, A), name);
  for (int trans = 0; trans < 2; ++trans) {
    must((trans ? oracle_hss_matvec_ranked_t : oracle_hss_matvec_ranked)(n, p, c, ranks, D, U, V, Rt, W, B, X, m, Y),
         name);
    dense_apply(n, A, X, m, R, trans);
    check(name, Y, R, n * m);
  }
  free(D); free(U); free(V); free(Rt); free(W); free(B); free(X); free(Y); free(R); free(A);
}

static void hss_noderanked_case(const char* name, int64_t n, int32_t p, const int64_t* c, const int32_t* kn,
                                int32_t m) {
  int64_t uv = 0, rw = 0, bb = 0;
  for (int64_t i = 0; i < (1ll << p); ++i) uv += leaf_rows(c, i) * kn[(1ll << p) - 2 + i];
  for (int l = 1; l < p; ++l)
    for (int64_t i = 0; i < (1ll << l); ++i) {
      const int64_t h = (1ll << l) - 2 + i, c0 = (1ll << (l + 1)) - 2 + 2 * i;
      rw += (int64_t)(kn[c0] + kn[c0 + 1]) * kn[h];
    }
  for (int l = 1; l <= p; ++l)
    for (int64_t q = 0; q < (1ll << (l - 1)); ++q) {
      const int64_t c0 = (1ll << l) - 2 + 2 * q;
      bb += 2ll * kn[c0] * kn[c0 + 1];
    }
  double *D = rnd(dblocks(c, p)), *U = rnd(uv), *V = rnd(uv), *Rt = rnd(rw), *W = rnd(rw), *B = rnd(bb),
         *X = rnd(n * m), *Y = rnd(n * m), *R = rnd(n * m), *A = rnd(n * n);
  must(oracle_hss_dense_noderanked(n, p, c, kn, D, U, V, Rt, W, B, A), name);
  for (int trans = 0; trans < 2; ++trans) {
    must((trans ? oracle_hss_matvec_noderanked_t : oracle_hss_matvec_noderanked)(n, p, c, kn, D, U, V, Rt, W, B, X, m,
                                                                                 Y),
         name);
    dense_apply(n, A, X, m, R, trans);
    check(name, Y, R, n * m);
  }
  free(D); free(U); free(V); free(Rt); free(W); free(B); free(X); free(Y); free(R); free(A);
}

int main(void) {
  /* uniform tree: n = 64, p = 3, leaf 8 */
  int64_t cu[8];
  for (int i = 0; i < 8; ++i) cu[i] = 8 * (i + 1);
  /* ragged tree with empty leaves: rows per leaf 5, 0, 9, 3, 0, 0, 11, 4 */
  const int64_t cr[8] = {5, 5, 14, 17, 17, 17, 28, 32};
  const int64_t c1[2] = {3, 7}, c0[1] = {6};
  const int32_t rk3[3] = {3, 0, 2}, rk1[1] = {2}, rku[3] = {2, 2, 2};
  for (int32_t m = 1; m <= 3; m += 2) {
    hodlr_case("hodlr uniform", 64, 3, cu, rk3, m);
    hodlr_case("hodlr ragged", 32, 3, cr, rk3, m);
    hodlr_case("hodlr ragged equal ranks", 32, 3, cr, rku, m);
    hodlr_case("hodlr p=1", 7, 1, c1, rk1, m);
    hodlr_case("hodlr p=0", 6, 0, c0, rk1, m);
    hss_case("hss uniform", 64, 3, cu, 3, m);
    hss_case("hss ragged", 32, 3, cr, 2, m);
    hss_case("hss p=1", 7, 1, c1, 2, m);
    hss_case("hss p=0", 6, 0, c0, 2, m);
    const int32_t hr[3] = {4, 2, 3}, hr0[3] = {3, 0, 2};
    hss_ranked_case("hss per-level ranks", 64, 3, cu, hr, m);
    hss_ranked_case("hss per-level ranks, rank-0 level", 32, 3, cr, hr0, m);
    /* node ranks, heap order: level 1 (2 nodes), level 2 (4), level 3 (8 leaves) */
    const int32_t kn[14] = {2, 3, 1, 0, 2, 3, 2, 1, 0, 3, 2, 2, 1, 3};
    hss_noderanked_case("hss per-node ranks", 64, 3, cu, kn, m);
    hss_noderanked_case("hss per-node ranks, ragged", 32, 3, cr, kn, m);
  }
  int32_t pd = 0;
  int64_t cd[64];
  must(oracle_default_cluster(100, 16, &pd, cd, 64), "default cluster");
  double* X = rnd(100 * 2);
  double* Y = rnd(100 * 2);
  must(oracle_laplacian_inverse_apply(100, X, 2, Y), "laplacian inverse");
  free(X); free(Y);
  if (g_fail) return 1;
  printf("oracle sanitize: clean\n");
  return 0;
}
