/*
 * hm_oracle.c — CPU ORACLE for Y = A X with A in HODLR or HSS format.
 *
 * TEST INFRASTRUCTURE ONLY (see hm_oracle.h). Plain, slow, obviously correct:
 * every routine follows the paper (hm-toolbox, arXiv 1909.07909,
 * /root/reference/PAPER.md, "P:n" = line n) in its own order and notation.
 * fp64 throughout (the paper's Matlab default, BASELINE.json fixes fp64);
 * every reduction is a sequential sum in natural index order, so the result
 * does not depend on the OpenMP thread count. Built with
 *   gcc -O2 -fno-fast-math -ffp-contract=off -fopenmp
 * (no FMA contraction, no reassociation).
 *
 * Parity status: every function here is pinned by tests/test_oracle_*.py
 * (dense brute force, closed forms, exact structured cases, invariants);
 * none is "parity unpinned".
 */
#include "hm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OMP_MIN_WORK 32768 /* only fork threads for loops doing at least this much */

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Thread count of the OpenMP loops (results do not depend on it: every
 * reduction is sequential in a fixed order). For the 1-thread / all-core
 * baseline rows of BASELINE.md §4. */
void oracle_set_num_threads(int n) {
#ifdef _OPENMP
  if (n >= 1) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* ---------------------------------------------------------------- trees -- */
/* Def. 2.1 + the leaf-endpoint vector c of P:560-565. */

static int check_tree(int64_t n, int32_t p, const int64_t* c) {
  if (n < 0 || p < 0 || p > 40 || c == NULL) return -1;
  int64_t nl = (int64_t)1 << p, prev = 0;
  for (int64_t i = 0; i < nl; ++i) {
    if (c[i] < prev) return -1; /* nondecreasing (Def. 2.1: n_0 <= n_1 <= ...) */
    prev = c[i];
  }
  return (c[nl - 1] == n) ? 0 : -1; /* n_{2^l} = n */
}

/* First row of leaf i: n_{i-1}^{(p)} (0 for the first leaf). */
static int64_t leaf_lo(const int64_t* c, int64_t i) { return i == 0 ? 0 : c[i - 1]; }

/* Row range of node (l, i): the union of its 2^(p-l) leaves (Def. 2.1: the
 * children form a partitioning of their parent). */
static void node_range(const int64_t* c, int32_t p, int32_t l, int64_t i, int64_t* lo, int64_t* hi) {
  int64_t span = (int64_t)1 << (p - l);
  *lo = leaf_lo(c, i * span);
  *hi = c[(i + 1) * span - 1];
}

/* Offset of leaf block D_i in the concatenated leaf array. */
static int64_t* leaf_block_offsets(const int64_t* c, int32_t p) {
  int64_t nl = (int64_t)1 << p;
  int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nl + 1));
  if (!off) return NULL;
  off[0] = 0;
  for (int64_t i = 0; i < nl; ++i) {
    int64_t s = c[i] - leaf_lo(c, i);
    off[i + 1] = off[i] + s * s;
  }
  return off;
}

int oracle_default_cluster(int64_t n, int64_t nmin, int32_t* p_out, int64_t* c_out, int64_t cap) {
  /* {1..n} -> {1..ceil(n/2)} u {ceil(n/2)+1..n}, repeated until the
   * minimal block size nmin is reached. Sets on one level have sizes
   * ceil(n/2^d) or less, so the depth is the least d with ceil(n/2^d) <= nmin. */
  if (n < 1 || nmin < 1 || p_out == NULL) return -1;
  int32_t p = 0;
  while (((n + ((int64_t)1 << p) - 1) >> p) > nmin) ++p;
  *p_out = p;
  if (c_out == NULL) return 0;
  int64_t nl = (int64_t)1 << p;
  if (cap < nl) return -1;
  /* level-by-level splitting of [lo, hi) into [lo, lo+ceil(s/2)), [.., hi) */
  int64_t* lo = (int64_t*)malloc(sizeof(int64_t) * (size_t)nl);
  int64_t* hi = (int64_t*)malloc(sizeof(int64_t) * (size_t)nl);
  if (!lo || !hi) { free(lo); free(hi); return -1; }
  lo[0] = 0; hi[0] = n;
  for (int32_t l = 0; l < p; ++l) {
    int64_t cnt = (int64_t)1 << l;
    for (int64_t i = cnt - 1; i >= 0; --i) { /* in place, back to front */
      int64_t a = lo[i], b = hi[i], s = b - a, h = (s + 1) / 2;
      lo[2 * i] = a;      hi[2 * i] = a + h;
      lo[2 * i + 1] = a + h; hi[2 * i + 1] = b;
    }
  }
  for (int64_t i = 0; i < nl; ++i) c_out[i] = hi[i];
  free(lo); free(hi);
  return 0;
}

/* ------------------------------------------------------ small products -- */

/* Y[r][:] = sum_j A[r][j] X[j][:]  (A: rows x cols row-major, lda; X: cols x m),
 * sums over j in natural order. Used for "if A is dense return Av"
 * and the diagonal blocks d_i = A(I_i,I_i) v(I_i). */
static void dense_mul(int64_t rows, int64_t cols, const double* A, int64_t lda,
                      const double* X, int32_t m, double* Y) {
#pragma omp parallel for schedule(static) if (rows * cols * m > OMP_MIN_WORK)
  for (int64_t r = 0; r < rows; ++r) {
    for (int32_t q = 0; q < m; ++q) {
      double s = 0.0;
      for (int64_t j = 0; j < cols; ++j) s += A[r * lda + j] * X[j * m + q];
      Y[r * m + q] = s;
    }
  }
}

/* Y[r][:] = sum_j A[j][r] X[j][:] — the product with A^T (A: cols x rows
 * row-major, lda), sums over j in natural order. The adjoint's leaf term
 * D_i^* v(I_i) (reading G4: * is the transpose). */
static void dense_mul_t(int64_t rows, int64_t cols, const double* A, int64_t lda,
                        const double* X, int32_t m, double* Y) {
#pragma omp parallel for schedule(static) if (rows * cols * m > OMP_MIN_WORK)
  for (int64_t r = 0; r < rows; ++r) {
    for (int32_t q = 0; q < m; ++q) {
      double s = 0.0;
      for (int64_t j = 0; j < cols; ++j) s += A[j * lda + r] * X[j * m + q];
      Y[r * m + q] = s;
    }
  }
}

/* t = V^T x : t[a][q] = sum_{r} V[r][a] x[r][q], rows in natural order
 * (the (V_j^{(l)})^* v(I_j) products of P:645-651 / P:686). V has ld = k. */
static void vt_mul(int64_t rows, int32_t k, const double* V, const double* X, int32_t m, double* t) {
#pragma omp parallel for collapse(2) schedule(static) if (rows * k * m > OMP_MIN_WORK)
  for (int32_t a = 0; a < k; ++a) {
    for (int32_t q = 0; q < m; ++q) {
      double s = 0.0;
      for (int64_t r = 0; r < rows; ++r) s += V[r * k + a] * X[r * m + q];
      t[a * m + q] = s;
    }
  }
}

/* ----------------------------------------------------------------- HODLR -- */

typedef struct {
  int64_t n;
  int32_t p;
  const int64_t* c;
  const int32_t* ranks;   /* ranks[l-1] = k_l, l = 1..p */
  int64_t* lvl_off;       /* offset of level l in U/V, l = 1..p (index l) */
  int64_t* d_off;         /* leaf block offsets */
  const double *D, *U, *V, *X;
  int32_t m;
  int trans;              /* 1: apply A^* (adjoint) */
  double* Y_out;
} hodlr_ctx;

/* A(I_a, I_b) v(I_b) for siblings a,b at level l, restricted to rows
 * [ra0, ra1) of I_a: y = U_l(rows) (V_l(I_b)^T v(I_b)) — the low-rank
 * off-diagonal product of Fig. 5 left, lines "y2 <- A12 v2", "y3 <- A21 v1". */
static int lowrank_apply(const hodlr_ctx* h, int32_t l, int64_t b_lo, int64_t b_hi,
                         int64_t ra0, int64_t ra1, double* y) {
  int32_t k = h->ranks[l - 1];
  int32_t m = h->m;
  int64_t rows = ra1 - ra0;
  if (k == 0) { /* rank 0 encodes the zero block ('eye'/'diagonal') */
    memset(y, 0, sizeof(double) * (size_t)(rows * m));
    return 0;
  }
  const double* Ul = h->U + h->lvl_off[l];
  const double* Vl = h->V + h->lvl_off[l];
  double* t = (double*)malloc(sizeof(double) * (size_t)k * (size_t)m);
  if (!t) return -1;
  vt_mul(b_hi - b_lo, k, Vl + b_lo * k, h->X + b_lo * m, m, t);
  dense_mul(rows, k, Ul + ra0 * k, k, t, m, y);
  free(t);
  return 0;
}

/* HODLR_matvec (Fig. 5 left) on node (l, i); writes Y(I_i^l). */
static int hodlr_rec(const hodlr_ctx* h, int32_t l, int64_t i) {
  int64_t lo, hi;
  node_range(h->c, h->p, l, i, &lo, &hi);
  int32_t m = h->m;
  if (l == h->p) { /* "if A is dense return Av" (A^* v for the adjoint) */
    int64_t s = hi - lo;
    if (h->trans) dense_mul_t(s, s, h->D + h->d_off[i], s, h->X + lo * m, m, h->Y_out + lo * m);
    else dense_mul(s, s, h->D + h->d_off[i], s, h->X + lo * m, m, h->Y_out + lo * m);
    return 0;
  }
  int64_t a = 2 * i, b = 2 * i + 1, alo, ahi, blo, bhi;
  node_range(h->c, h->p, l + 1, a, &alo, &ahi);
  node_range(h->c, h->p, l + 1, b, &blo, &bhi);
  /* y1 <- HODLR_matvec(A11, v1), stored directly in Y(I_a) */
  if (hodlr_rec(h, l + 1, a)) return -1;
  /* y2 <- A12 v2 ; y3 <- A21 v1 */
  double* y2 = (double*)malloc(sizeof(double) * (size_t)((ahi - alo) * m + 1));
  double* y3 = (double*)malloc(sizeof(double) * (size_t)((bhi - blo) * m + 1));
  if (!y2 || !y3) { free(y2); free(y3); return -1; }
  if (lowrank_apply(h, l + 1, blo, bhi, alo, ahi, y2)) return -1;
  if (lowrank_apply(h, l + 1, alo, ahi, blo, bhi, y3)) return -1;
  /* y4 <- HODLR_matvec(A22, v2), stored directly in Y(I_b) */
  if (hodlr_rec(h, l + 1, b)) return -1;
  /* return [y1 + y2; y3 + y4] */
  for (int64_t e = 0; e < (ahi - alo) * m; ++e) h->Y_out[alo * m + e] = h->Y_out[alo * m + e] + y2[e];
  for (int64_t e = 0; e < (bhi - blo) * m; ++e) h->Y_out[blo * m + e] = y3[e] + h->Y_out[blo * m + e];
  free(y2); free(y3);
  return 0;
}

static int hodlr_setup(hodlr_ctx* h, int64_t n, int32_t p, const int64_t* c, const int32_t* ranks,
                       const double* D, const double* U, const double* V, const double* X, int32_t m) {
  memset(h, 0, sizeof(*h));
  if (check_tree(n, p, c) || m < 1 || (p > 0 && ranks == NULL)) return -1;
  for (int32_t l = 1; l <= p; ++l)
    if (ranks[l - 1] < 0) return -1;
  h->n = n; h->p = p; h->c = c; h->ranks = ranks;
  h->D = D; h->U = U; h->V = V; h->X = X; h->m = m;
  h->lvl_off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(p + 2));
  h->d_off = leaf_block_offsets(c, p);
  if (!h->lvl_off || !h->d_off) return -1;
  h->lvl_off[0] = 0;
  h->lvl_off[1] = 0;
  for (int32_t l = 1; l <= p; ++l) h->lvl_off[l + 1] = h->lvl_off[l] + n * (int64_t)ranks[l - 1];
  return 0;
}

static void hodlr_teardown(hodlr_ctx* h) {
  free(h->lvl_off);
  free(h->d_off);
}

/* The adjoint A^* of a HODLR matrix is a HODLR matrix on the same tree:
 * A^*(I_a, I_b) = (A(I_b, I_a))^* = (U_l(I_b) V_l(I_a)^*)^* = V_l(I_a) U_l(I_b)^*
 * for siblings a, b (Def. 2.2), and A^*(I_i, I_i) = D_i^*. So the
 * adjoint product is Fig. 5 left with the roles of U and V exchanged and the
 * leaf blocks transposed (P:404, P:416 use A^* products). */
static int hodlr_matvec_op(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks,
                           const double* D, const double* U, const double* V,
                           const double* X, int32_t m, double* Y, int trans) {
  hodlr_ctx h;
  if (hodlr_setup(&h, n, p, c, ranks, D, trans ? V : U, trans ? U : V, X, m) || Y == NULL) {
    hodlr_teardown(&h);
    return -1;
  }
  h.trans = trans;
  h.Y_out = Y;
  int rc = hodlr_rec(&h, 0, 0);
  hodlr_teardown(&h);
  return rc;
}

static int hodlr_matvec_leaves_op(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks,
                                  const double* Dsel, const double* U, const double* V,
                                  const double* X, int32_t m,
                                  const int64_t* leaves, int64_t nleaves, double* Yout, int trans) {
  /* The recursion of Fig. 5 left, followed only down the root-to-leaf path of
   * each listed leaf. On that path, the rows of leaf L receive, in the
   * recursion's order: the leaf product D_L v(I_L) ("if A is dense return
   * Av"), then on the way back up, level by level l = p..1, the off-diagonal
   * term U_l(I_L) (V_l(I_sib)^T v(I_sib)) of the block coupling the level-l
   * node on the path with its sibling ("y1 + y2" / "y3 + y4"). */
  hodlr_ctx h;
  if (hodlr_setup(&h, n, p, c, ranks, NULL, trans ? V : U, trans ? U : V, X, m) || Yout == NULL ||
      leaves == NULL) {
    hodlr_teardown(&h);
    return -1;
  }
  int64_t nl = (int64_t)1 << p, yoff = 0, doff = 0;
  int rc = 0;
  for (int64_t s = 0; s < nleaves && rc == 0; ++s) {
    int64_t L = leaves[s];
    if (L < 0 || L >= nl) { rc = -1; break; }
    int64_t lo = leaf_lo(c, L), hi = c[L], rows = hi - lo;
    double* y = Yout + yoff;
    if (trans) dense_mul_t(rows, rows, Dsel + doff, rows, X + lo * m, m, y);
    else dense_mul(rows, rows, Dsel + doff, rows, X + lo * m, m, y);
    double* term = (double*)malloc(sizeof(double) * (size_t)(rows * m + 1));
    if (!term) { rc = -1; break; }
    for (int32_t l = p; l >= 1; --l) {
      int64_t node = L >> (p - l), sib = node ^ 1, slo, shi;
      node_range(c, p, l, sib, &slo, &shi);
      if (lowrank_apply(&h, l, slo, shi, lo, hi, term)) { rc = -1; break; }
      for (int64_t e = 0; e < rows * m; ++e) y[e] = y[e] + term[e];
    }
    free(term);
    yoff += rows * m;
    doff += rows * rows;
  }
  hodlr_teardown(&h);
  return rc;
}

int oracle_hodlr_matvec(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks,
                        const double* D, const double* U, const double* V,
                        const double* X, int32_t m, double* Y) {
  return hodlr_matvec_op(n, p, c, ranks, D, U, V, X, m, Y, 0);
}

int oracle_hodlr_matvec_t(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks,
                          const double* D, const double* U, const double* V,
                          const double* X, int32_t m, double* Y) {
  return hodlr_matvec_op(n, p, c, ranks, D, U, V, X, m, Y, 1);
}

int oracle_hodlr_matvec_leaves(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks,
                               const double* Dsel, const double* U, const double* V,
                               const double* X, int32_t m,
                               const int64_t* leaves, int64_t nleaves, double* Yout) {
  return hodlr_matvec_leaves_op(n, p, c, ranks, Dsel, U, V, X, m, leaves, nleaves, Yout, 0);
}

int oracle_hodlr_matvec_t_leaves(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks,
                                 const double* Dsel, const double* U, const double* V,
                                 const double* X, int32_t m,
                                 const int64_t* leaves, int64_t nleaves, double* Yout) {
  return hodlr_matvec_leaves_op(n, p, c, ranks, Dsel, U, V, X, m, leaves, nleaves, Yout, 1);
}

int oracle_hodlr_dense(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks,
                       const double* D, const double* U, const double* V, double* A) {
  /* Def. 2.2: A(I_i^p, I_i^p) = D_i; every sibling off-diagonal
   * block A(I_a^l, I_b^l), l = 1..p, equals U_l(I_a) V_l(I_b)^T. */
  hodlr_ctx h;
  if (hodlr_setup(&h, n, p, c, ranks, D, U, V, NULL, 1) || A == NULL) { hodlr_teardown(&h); return -1; }
  memset(A, 0, sizeof(double) * (size_t)(n * n));
  int64_t nl = (int64_t)1 << p;
  for (int64_t i = 0; i < nl; ++i) {
    int64_t lo = leaf_lo(c, i), s = c[i] - lo;
    for (int64_t r = 0; r < s; ++r)
      for (int64_t q = 0; q < s; ++q) A[(lo + r) * n + lo + q] = D[h.d_off[i] + r * s + q];
  }
  for (int32_t l = 1; l <= p; ++l) {
    int32_t k = ranks[l - 1];
    const double* Ul = U + h.lvl_off[l];
    const double* Vl = V + h.lvl_off[l];
    for (int64_t a = 0; a < ((int64_t)1 << l); ++a) {
      int64_t b = a ^ 1, alo, ahi, blo, bhi;
      node_range(c, p, l, a, &alo, &ahi);
      node_range(c, p, l, b, &blo, &bhi);
      for (int64_t r = alo; r < ahi; ++r)
        for (int64_t q = blo; q < bhi; ++q) {
          double s = 0.0;
          for (int32_t e = 0; e < k; ++e) s += Ul[r * k + e] * Vl[q * k + e];
          A[r * n + q] = s;
        }
    }
  }
  hodlr_teardown(&h);
  return 0;
}

/* ------------------------------------------------------------------- HSS -- */
/* Ranks may differ per node (bases and translation operators need not
 * have k columns "for every level and node ... as long as the dimensions are
 * compatible"). Node (l, i), l = 1..p, has rank k_h at heap index
 * h = 2^l - 2 + i. Then U_i^(p), V_i^(p) are |I_i| x k_h, the translations
 * R_{U,i}^(l), R_{V,i}^(l) are (k_{2i} + k_{2i+1}) x k_h (eq. (3) P:256-259 with
 * the children's columns), the cores of siblings 2q, 2q+1 are
 * S_{2q,2q+1}: k_{2q} x k_{2q+1} and S_{2q+1,2q}: k_{2q+1} x k_{2q}, and the
 * coefficient vectors v_i^l are k_h x m. Flat layout (row-major, heap order;
 * the per-level and uniform layouts of hm.h are special cases):
 *   U, V  leaf after leaf: leaf i's |I_i| x k rows
 *   R, W  node (l, i), l = 1..p-1, heap order: [k_{2i} + k_{2i+1}][k_h]
 *   B     parent (l-1, q), l = 1..p, heap order from the root: B12 then B21 */

typedef struct {
  int64_t n;
  int32_t p, m;
  const int64_t* c;
  int64_t* d_off;
  int32_t* kn;      /* kn[h] = rank of node h = 2^l - 2 + i (l >= 1) */
  int64_t* cf_off;  /* coefficient block of node h in xh / yh, in doubles */
  int64_t* rw_off;  /* R / W of node h (l = 1..p-1) */
  int64_t* b_off;   /* cores of the children of parent hp = 2^(l-1) - 1 + q (root hp = 0) */
  int64_t* u_off;   /* U / V rows of leaf i */
  const double *D, *U, *V, *R, *W, *B, *X;
  double* xh; /* v_i^l of Step 1, one k_h x m block per node */
  double* yh; /* the same vectors after Steps 2-3 */
  int trans;  /* 1: apply A^* (adjoint), see hss_matvec_op */
} hss_ctx;

static int64_t hidx(int32_t l, int64_t i) { return ((int64_t)1 << l) - 2 + i; }
static int32_t kof(const hss_ctx* s, int32_t l, int64_t i) { return l >= 1 ? s->kn[hidx(l, i)] : 0; }

static double* coef(const hss_ctx* s, double* base, int32_t l, int64_t i) {
  return base + s->cf_off[hidx(l, i)];
}

/* node_ranks: heap order, 2^(p+1) - 2 entries (nodes of levels 1..p) */
static int hss_setup(hss_ctx* s, int64_t n, int32_t p, const int64_t* c, const int32_t* node_ranks,
                     const double* D, const double* U, const double* V,
                     const double* R, const double* W, const double* B, const double* X, int32_t m) {
  memset(s, 0, sizeof(*s));
  if (check_tree(n, p, c) || m < 1 || (p > 0 && node_ranks == NULL)) return -1;
  s->n = n; s->p = p; s->m = m; s->c = c;
  s->D = D; s->U = U; s->V = V; s->R = R; s->W = W; s->B = B; s->X = X;
  s->d_off = leaf_block_offsets(c, p);
  const int64_t nn = ((int64_t)1 << (p + 1)) - 2, nl = (int64_t)1 << p;
  s->kn = (int32_t*)calloc((size_t)(nn + 1), sizeof(int32_t));
  s->cf_off = (int64_t*)calloc((size_t)(nn + 1), sizeof(int64_t));
  s->rw_off = (int64_t*)calloc((size_t)(nn + 1), sizeof(int64_t));
  s->b_off = (int64_t*)calloc((size_t)(nn + 1), sizeof(int64_t));
  s->u_off = (int64_t*)calloc((size_t)(nl + 1), sizeof(int64_t));
  if (!s->d_off || !s->kn || !s->cf_off || !s->rw_off || !s->b_off || !s->u_off) return -1;
  for (int64_t h = 0; h < nn; ++h) {
    if (node_ranks[h] < 0) return -1;
    s->kn[h] = node_ranks[h];
  }
  int64_t cf = 0, rw = 0, bo = 0;
  for (int32_t l = 1; l <= p; ++l)
    for (int64_t i = 0; i < ((int64_t)1 << l); ++i) {
      s->cf_off[hidx(l, i)] = cf;
      cf += (int64_t)kof(s, l, i) * m;
      if (l <= p - 1) {
        s->rw_off[hidx(l, i)] = rw;
        rw += (int64_t)(kof(s, l + 1, 2 * i) + kof(s, l + 1, 2 * i + 1)) * kof(s, l, i);
      }
    }
  for (int32_t l = 1; l <= p; ++l) /* parents (l-1, q) in heap order from the root */
    for (int64_t q = 0; q < ((int64_t)1 << (l - 1)); ++q) {
      s->b_off[((int64_t)1 << (l - 1)) - 1 + q] = bo;
      bo += 2 * (int64_t)kof(s, l, 2 * q) * kof(s, l, 2 * q + 1);
    }
  for (int64_t i = 0; i < nl; ++i)
    s->u_off[i + 1] = s->u_off[i] + (c[i] - leaf_lo(c, i)) * (int64_t)(p > 0 ? kof(s, p, i) : 0);
  size_t cnt = (size_t)cf + 1;
  s->xh = (double*)calloc(cnt, sizeof(double));
  s->yh = (double*)calloc(cnt, sizeof(double));
  return (s->xh && s->yh) ? 0 : -1;
}

static void hss_teardown(hss_ctx* s) {
  free(s->d_off); free(s->xh); free(s->yh);
  free(s->kn); free(s->cf_off); free(s->rw_off); free(s->b_off); free(s->u_off);
}

/* Step 1, first half, and the upsweep (Fig. 5 right):
 *   v_i^p = (V_i^(p))^* v(I_i^p),  i = 1..2^p
 *   v_i^l = (R_{V,i}^(l))^* [v_{2i-1}^{l+1}; v_{2i}^{l+1}],  l = p-1..1
 * with R_{V,i}^(l) = W[node] = [Wl; Wr] ((k_{2i} + k_{2i+1}) x k_h), reading G3. */
static void hss_upsweep(hss_ctx* s) {
  int32_t p = s->p, m = s->m;
  if (p == 0) return;
  int64_t nl = (int64_t)1 << p;
#pragma omp parallel for schedule(static) if (s->n * m * 16 > OMP_MIN_WORK)
  for (int64_t i = 0; i < nl; ++i) {
    int64_t lo = leaf_lo(s->c, i), hi = s->c[i];
    int32_t kp = kof(s, p, i);
    const double* Vi = s->V + s->u_off[i];  /* rows lo..hi-1 of leaf i, kp columns */
    double* t = coef(s, s->xh, p, i);
    for (int32_t a = 0; a < kp; ++a)
      for (int32_t q = 0; q < m; ++q) {
        double acc = 0.0;
        for (int64_t r = lo; r < hi; ++r) acc += Vi[(r - lo) * kp + a] * s->X[r * m + q];
        t[a * m + q] = acc;
      }
  }
  for (int32_t l = p - 1; l >= 1; --l) {
    int64_t cnt = (int64_t)1 << l;
#pragma omp parallel for schedule(static) if (cnt * 64 * m > OMP_MIN_WORK)
    for (int64_t i = 0; i < cnt; ++i) {
      int32_t k = kof(s, l, i), k0 = kof(s, l + 1, 2 * i), k1 = kof(s, l + 1, 2 * i + 1);
      const double* Wn = s->W + s->rw_off[hidx(l, i)]; /* [k0 + k1][k] */
      const double* z0 = coef(s, s->xh, l + 1, 2 * i);     /* v_{2i-1}^{l+1} */
      const double* z1 = coef(s, s->xh, l + 1, 2 * i + 1); /* v_{2i}^{l+1}   */
      double* t = coef(s, s->xh, l, i);
      for (int32_t a = 0; a < k; ++a)
        for (int32_t q = 0; q < m; ++q) {
          double acc = 0.0; /* (W^T z)[a] = sum_r W[r][a] z[r], r in natural order */
          for (int32_t r = 0; r < k0; ++r) acc += Wn[r * k + a] * z0[r * m + q];
          for (int32_t r = 0; r < k1; ++r) acc += Wn[(k0 + r) * k + a] * z1[r * m + q];
          t[a * m + q] = acc;
        }
    }
  }
}

/* Step 2 for one sibling pair (reading G1: l = 1..p, q = 0..2^(l-1)-1):
 *   [v_{2q}^l; v_{2q+1}^l] <- [0 S_{2q,2q+1}; S_{2q+1,2q} 0] [v_{2q}^l; v_{2q+1}^l]
 * S_{2q,2q+1}^{(l)} = B12 (k_{2q} x k_{2q+1}) and S_{2q+1,2q}^{(l)} = B21 of the
 * parent (l-1, q). Writes only the member `which` (0 = 2q, 1 = 2q+1). */
static void hss_couple(hss_ctx* s, int32_t l, int64_t q, int which) {
  int32_t m = s->m, k0 = kof(s, l, 2 * q), k1 = kof(s, l, 2 * q + 1);
  const double* Bn = s->B + s->b_off[((int64_t)1 << (l - 1)) - 1 + q];
  const double* B12 = Bn;                     /* k0 x k1 */
  const double* B21 = Bn + (int64_t)k0 * k1;  /* k1 x k0 */
  const double* xin = coef(s, s->xh, l, 2 * q + (which == 0 ? 1 : 0));
  double* yout = coef(s, s->yh, l, 2 * q + which);
  int32_t ko = which == 0 ? k0 : k1, ki = which == 0 ? k1 : k0; /* output / input rank */
  /* A: S = B12 (which 0) or B21 (which 1), [ko][ki]. A^*: the cores of A^* are
   * S'_{2q,2q+1} = (S_{2q+1,2q})^* = B21^T and S'_{2q+1,2q} = B12^T; B21^T is
   * (k1 x k0)^T = k0 x k1, read transposed from B21. */
  for (int32_t a = 0; a < ko; ++a)
    for (int32_t c2 = 0; c2 < m; ++c2) {
      double acc = 0.0;
      for (int32_t r = 0; r < ki; ++r) {
        double sv;
        if (s->trans) sv = which == 0 ? B21[r * k0 + a] : B12[r * k1 + a];
        else sv = which == 0 ? B12[a * k1 + r] : B21[a * k0 + r];
        acc += sv * xin[r * m + c2];
      }
      yout[a * m + c2] = acc;
    }
}

/* Step 3 for one child:
 *   [v_{2i-1}^{l+1}; v_{2i}^{l+1}] <- [v_{2i-1}^{l+1}; v_{2i}^{l+1}] + R_{U,i}^{(l)} v_i^l
 * R_{U,i}^{(l)} = R[node] = [Rl; Rr] ((k_{2i} + k_{2i+1}) x k_h). Updates child `which`. */
static void hss_down(hss_ctx* s, int32_t l, int64_t i, int which) {
  int32_t k = kof(s, l, i), k0 = kof(s, l + 1, 2 * i), m = s->m;
  int32_t kc = kof(s, l + 1, 2 * i + which);
  const double* Rn = s->R + s->rw_off[hidx(l, i)] + (which == 0 ? 0 : (int64_t)k0 * k);
  const double* yin = coef(s, s->yh, l, i);
  double* ych = coef(s, s->yh, l + 1, 2 * i + which);
  for (int32_t a = 0; a < kc; ++a)
    for (int32_t c2 = 0; c2 < m; ++c2) {
      double acc = 0.0;
      for (int32_t r = 0; r < k; ++r) acc += Rn[a * k + r] * yin[r * m + c2];
      ych[a * m + c2] = ych[a * m + c2] + acc;
    }
}

/* Step 4 for one leaf (reading G2): y(I_i) = U_i v_i^p + d_i,
 * d_i = A(I_i, I_i) v(I_i). Dblk is D_i, y the leaf's output rows. */
static void hss_leaf_out(const hss_ctx* s, int64_t i, const double* Dblk, double* y) {
  int32_t m = s->m, p = s->p;
  int32_t k = p > 0 ? kof(s, p, i) : 0;
  int64_t lo = leaf_lo(s->c, i), rows = s->c[i] - lo;
  const double* yv = (p > 0 && k > 0) ? coef(s, s->yh, p, i) : NULL;
  const double* Ui = p > 0 ? s->U + s->u_off[i] : NULL;
  for (int64_t r = 0; r < rows; ++r)
    for (int32_t q = 0; q < m; ++q) {
      double d = 0.0;
      for (int64_t j = 0; j < rows; ++j)
        d += (s->trans ? Dblk[j * rows + r] : Dblk[r * rows + j]) * s->X[(lo + j) * m + q];
      double u = 0.0;
      if (yv)
        for (int32_t a = 0; a < k; ++a) u += Ui[r * k + a] * yv[a * m + q];
      y[r * m + q] = u + d;
    }
}

/* Steps 2 and 3 on every node (the whole tree). */
static void hss_couple_down_all(hss_ctx* s) {
  int32_t p = s->p;
  for (int32_t l = 1; l <= p; ++l) { /* Step 2, all levels incl. the leaves (G1) */
    int64_t pairs = (int64_t)1 << (l - 1);
#pragma omp parallel for schedule(static) if (pairs * 64 * s->m > OMP_MIN_WORK)
    for (int64_t q = 0; q < pairs; ++q) {
      hss_couple(s, l, q, 0);
      hss_couple(s, l, q, 1);
    }
  }
  for (int32_t l = 1; l <= p - 1; ++l) { /* Step 3, top to bottom */
    int64_t cnt = (int64_t)1 << l;
#pragma omp parallel for schedule(static) if (cnt * 64 * s->m > OMP_MIN_WORK)
    for (int64_t i = 0; i < cnt; ++i) {
      hss_down(s, l, i, 0);
      hss_down(s, l, i, 1);
    }
  }
}

/* The adjoint of an HSS matrix is HSS on the same tree (eq. (3)):
 * A^*(I_b, I_a) = (U_a^(l) S_ab V_b^(l)*)^* = V_b^(l) S_ab^* U_a^(l)*, so A^*
 * has row bases V (translations W), column bases U (translations R), cores
 * S'_ba = S_ab^* and leaf blocks D_i^*. hss_matvec_op runs Fig. 5 right on
 * those generators (trans = 1): U <-> V and R <-> W exchanged here, the
 * transposed cores in hss_couple, D_i^* in hss_leaf_out. */
static int hss_matvec_op(int64_t n, int32_t p, const int64_t* c, const int32_t* node_ranks,
                         const double* D, const double* U, const double* V,
                         const double* R, const double* W, const double* B,
                         const double* X, int32_t m, double* Y, int trans) {
  hss_ctx s;
  if (hss_setup(&s, n, p, c, node_ranks, D, trans ? V : U, trans ? U : V, trans ? W : R, trans ? R : W, B, X, m) ||
      Y == NULL) {
    hss_teardown(&s);
    return -1;
  }
  s.trans = trans;
  hss_upsweep(&s);
  hss_couple_down_all(&s);
  int64_t nl = (int64_t)1 << p;
#pragma omp parallel for schedule(dynamic, 1) if (n * m * 8 > OMP_MIN_WORK)
  for (int64_t i = 0; i < nl; ++i)
    hss_leaf_out(&s, i, D + s.d_off[i], Y + leaf_lo(c, i) * m);
  hss_teardown(&s);
  return 0;
}

static int hss_matvec_leaves_op(int64_t n, int32_t p, const int64_t* c, const int32_t* node_ranks,
                                const double* Dsel, const double* U, const double* V,
                                const double* R, const double* W, const double* B,
                                const double* X, int32_t m,
                                const int64_t* leaves, int64_t nleaves, double* Yout, int trans) {
  hss_ctx s;
  if (hss_setup(&s, n, p, c, node_ranks, NULL, trans ? V : U, trans ? U : V, trans ? W : R, trans ? R : W, B, X,
                m) ||
      Yout == NULL || leaves == NULL) {
    hss_teardown(&s);
    return -1;
  }
  s.trans = trans;
  hss_upsweep(&s); /* every v_i^l is needed: couplings read siblings' vectors */
  int64_t nl = (int64_t)1 << p, yoff = 0, doff = 0;
  for (int64_t t = 0; t < nleaves; ++t) {
    int64_t L = leaves[t];
    if (L < 0 || L >= nl) { hss_teardown(&s); return -1; }
    /* Step 2 on the path nodes (l, L >> (p-l)), l = 1..p, then Step 3 along it */
    for (int32_t l = 1; l <= p; ++l) {
      int64_t node = L >> (p - l);
      hss_couple(&s, l, node >> 1, (int)(node & 1));
    }
    for (int32_t l = 1; l <= p - 1; ++l) {
      int64_t node = L >> (p - l), child = L >> (p - l - 1);
      hss_down(&s, l, node, (int)(child & 1));
    }
    int64_t rows = c[L] - leaf_lo(c, L);
    hss_leaf_out(&s, L, Dsel + doff, Yout + yoff);
    yoff += rows * m;
    doff += rows * rows;
  }
  hss_teardown(&s);
  return 0;
}

/* Per-node rank arrays (heap order, levels 1..p) of the uniform (k) and
 * per-level (ranks[l-1] = k_l) entry points. */
static int32_t* node_ranks_of_levels(int32_t p, const int32_t* ranks, int32_t k) {
  const int64_t nn = ((int64_t)1 << (p + 1)) - 2;
  int32_t* r = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nn + 1));
  if (!r) return NULL;
  for (int32_t l = 1; l <= p; ++l)
    for (int64_t i = 0; i < ((int64_t)1 << l); ++i) r[((int64_t)1 << l) - 2 + i] = ranks ? ranks[l - 1] : k;
  return r;
}

int oracle_hss_matvec(int64_t n, int32_t p, const int64_t* c, int32_t k,
                      const double* D, const double* U, const double* V,
                      const double* R, const double* W, const double* B,
                      const double* X, int32_t m, double* Y) {
  if (k < 0 || p < 0 || p > 40) return -1;
  int32_t* r = node_ranks_of_levels(p, NULL, k);
  int rc = r ? hss_matvec_op(n, p, c, r, D, U, V, R, W, B, X, m, Y, 0) : -1;
  free(r);
  return rc;
}

int oracle_hss_matvec_t(int64_t n, int32_t p, const int64_t* c, int32_t k,
                        const double* D, const double* U, const double* V,
                        const double* R, const double* W, const double* B,
                        const double* X, int32_t m, double* Y) {
  if (k < 0 || p < 0 || p > 40) return -1;
  int32_t* r = node_ranks_of_levels(p, NULL, k);
  int rc = r ? hss_matvec_op(n, p, c, r, D, U, V, R, W, B, X, m, Y, 1) : -1;
  free(r);
  return rc;
}

static int hss_ranked_op(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks,
                         const double* D, const double* U, const double* V, const double* R, const double* W,
                         const double* B, const double* X, int32_t m, double* Y, int trans) {
  if (p < 0 || p > 40 || (p > 0 && !ranks)) return -1;
  int32_t* r = node_ranks_of_levels(p, ranks, 0);
  int rc = r ? hss_matvec_op(n, p, c, r, D, U, V, R, W, B, X, m, Y, trans) : -1;
  free(r);
  return rc;
}

int oracle_hss_matvec_ranked(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks,
                             const double* D, const double* U, const double* V,
                             const double* R, const double* W, const double* B,
                             const double* X, int32_t m, double* Y) {
  return hss_ranked_op(n, p, c, ranks, D, U, V, R, W, B, X, m, Y, 0);
}

int oracle_hss_matvec_ranked_t(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks,
                               const double* D, const double* U, const double* V,
                               const double* R, const double* W, const double* B,
                               const double* X, int32_t m, double* Y) {
  return hss_ranked_op(n, p, c, ranks, D, U, V, R, W, B, X, m, Y, 1);
}

int oracle_hss_matvec_noderanked(int64_t n, int32_t p, const int64_t* c, const int32_t* node_ranks,
                                 const double* D, const double* U, const double* V,
                                 const double* R, const double* W, const double* B,
                                 const double* X, int32_t m, double* Y) {
  return hss_matvec_op(n, p, c, node_ranks, D, U, V, R, W, B, X, m, Y, 0);
}

int oracle_hss_matvec_noderanked_t(int64_t n, int32_t p, const int64_t* c, const int32_t* node_ranks,
                                   const double* D, const double* U, const double* V,
                                   const double* R, const double* W, const double* B,
                                   const double* X, int32_t m, double* Y) {
  return hss_matvec_op(n, p, c, node_ranks, D, U, V, R, W, B, X, m, Y, 1);
}

int oracle_hss_matvec_leaves(int64_t n, int32_t p, const int64_t* c, int32_t k,
                             const double* Dsel, const double* U, const double* V,
                             const double* R, const double* W, const double* B,
                             const double* X, int32_t m,
                             const int64_t* leaves, int64_t nleaves, double* Yout) {
  if (k < 0 || p < 0 || p > 40) return -1;
  int32_t* r = node_ranks_of_levels(p, NULL, k);
  int rc = r ? hss_matvec_leaves_op(n, p, c, r, Dsel, U, V, R, W, B, X, m, leaves, nleaves, Yout, 0) : -1;
  free(r);
  return rc;
}

int oracle_hss_matvec_t_leaves(int64_t n, int32_t p, const int64_t* c, int32_t k,
                               const double* Dsel, const double* U, const double* V,
                               const double* R, const double* W, const double* B,
                               const double* X, int32_t m,
                               const int64_t* leaves, int64_t nleaves, double* Yout) {
  if (k < 0 || p < 0 || p > 40) return -1;
  int32_t* r = node_ranks_of_levels(p, NULL, k);
  int rc = r ? hss_matvec_leaves_op(n, p, c, r, Dsel, U, V, R, W, B, X, m, leaves, nleaves, Yout, 1) : -1;
  free(r);
  return rc;
}

int oracle_hss_dense_noderanked(int64_t n, int32_t p, const int64_t* c, const int32_t* node_ranks,
                                const double* D, const double* U, const double* V,
                                const double* R, const double* W, const double* B, double* A) {
  /* Definition: diagonal leaf blocks D_i; every sibling block
   * A(I_a^l, I_b^l) = U_a^(l) S_ab^(l) (V_b^(l))^T, with the bases
   * of the upper levels rebuilt from the leaf bases by eq. (3):
   *   U_i^(l) = blockdiag(U_{2i}^(l+1), U_{2i+1}^(l+1)) R_{U,i}^(l), same for V
   * with R_{V,i}^(l) = W[node]; k_h columns on node h. */
  hss_ctx s;
  if (A == NULL || hss_setup(&s, n, p, c, node_ranks, D, U, V, R, W, B, NULL, 1)) { hss_teardown(&s); return -1; }
  memset(A, 0, sizeof(double) * (size_t)(n * n));
  int64_t nl = (int64_t)1 << p;
  for (int64_t i = 0; i < nl; ++i) {
    int64_t lo = leaf_lo(c, i), sz = c[i] - lo;
    for (int64_t r = 0; r < sz; ++r)
      for (int64_t q = 0; q < sz; ++q) A[(lo + r) * n + lo + q] = D[s.d_off[i] + r * sz + q];
  }
  if (p == 0) { hss_teardown(&s); return 0; }
  /* Ub, Vb: node h's basis (|I_h| x k_h rows, row-major) at bo[h] */
  const int64_t nn = ((int64_t)1 << (p + 1)) - 2;
  int64_t* bo = (int64_t*)calloc((size_t)(nn + 1), sizeof(int64_t));
  int64_t tot = 0, kmax = 1;
  for (int32_t l = 1; l <= p; ++l)
    for (int64_t i = 0; i < ((int64_t)1 << l); ++i) {
      int64_t lo, hi;
      node_range(c, p, l, i, &lo, &hi);
      bo[hidx(l, i)] = tot;
      tot += (hi - lo) * (int64_t)kof(&s, l, i);
      kmax = kof(&s, l, i) > kmax ? kof(&s, l, i) : kmax;
    }
  double* Ub = (double*)calloc((size_t)(tot + 1), sizeof(double));
  double* Vb = (double*)calloc((size_t)(tot + 1), sizeof(double));
  double* tmp = (double*)malloc(sizeof(double) * (size_t)(kmax + 1));
  if (!Ub || !Vb || !bo || !tmp) { free(Ub); free(Vb); free(bo); free(tmp); hss_teardown(&s); return -1; }
  for (int64_t i = 0; i < nl; ++i) { /* leaf bases */
    int64_t cnt = s.u_off[i + 1] - s.u_off[i];
    memcpy(Ub + bo[hidx(p, i)], U + s.u_off[i], sizeof(double) * (size_t)cnt);
    memcpy(Vb + bo[hidx(p, i)], V + s.u_off[i], sizeof(double) * (size_t)cnt);
  }
  for (int32_t l = p - 1; l >= 1; --l)
    for (int64_t i = 0; i < ((int64_t)1 << l); ++i) {
      int32_t k = kof(&s, l, i), k0 = kof(&s, l + 1, 2 * i);
      int64_t lo, hi;
      node_range(c, p, l, i, &lo, &hi);
      for (int ch = 0; ch < 2; ++ch) {
        int32_t kc = kof(&s, l + 1, 2 * i + ch);
        int64_t clo, chi;
        node_range(c, p, l + 1, 2 * i + ch, &clo, &chi);
        const double* Rh = R + s.rw_off[hidx(l, i)] + (ch ? (int64_t)k0 * k : 0); /* kc x k */
        const double* Wh = W + s.rw_off[hidx(l, i)] + (ch ? (int64_t)k0 * k : 0);
        const double* Uc = Ub + bo[hidx(l + 1, 2 * i + ch)];
        const double* Vc = Vb + bo[hidx(l + 1, 2 * i + ch)];
        for (int64_t r = clo; r < chi; ++r)
          for (int32_t a = 0; a < k; ++a) {
            double su = 0.0, sv = 0.0;
            for (int32_t e = 0; e < kc; ++e) {
              su += Uc[(r - clo) * kc + e] * Rh[e * k + a];
              sv += Vc[(r - clo) * kc + e] * Wh[e * k + a];
            }
            Ub[bo[hidx(l, i)] + (r - lo) * k + a] = su;
            Vb[bo[hidx(l, i)] + (r - lo) * k + a] = sv;
          }
      }
    }
  for (int32_t l = 1; l <= p; ++l)
    for (int64_t q = 0; q < ((int64_t)1 << (l - 1)); ++q) {
      const int32_t k0 = kof(&s, l, 2 * q), k1 = kof(&s, l, 2 * q + 1);
      const double* Bn = B + s.b_off[((int64_t)1 << (l - 1)) - 1 + q];
      for (int w = 0; w < 2; ++w) { /* w=0: A(I_2q, I_2q+1) = U S12 V^T; w=1: A(I_2q+1, I_2q) */
        int64_t a = 2 * q + w, b = 2 * q + 1 - w, alo, ahi, blo, bhi;
        node_range(c, p, l, a, &alo, &ahi);
        node_range(c, p, l, b, &blo, &bhi);
        const int32_t ka = w ? k1 : k0, kb = w ? k0 : k1;
        const double* S = Bn + (w ? (int64_t)k0 * k1 : 0); /* ka x kb */
        const double* Ua = Ub + bo[hidx(l, a)];
        const double* Vbb = Vb + bo[hidx(l, b)];
        for (int64_t r = alo; r < ahi; ++r) {
          for (int32_t e = 0; e < kb; ++e) { /* (U_a S)[r][e] */
            double su = 0.0;
            for (int32_t f = 0; f < ka; ++f) su += Ua[(r - alo) * ka + f] * S[f * kb + e];
            tmp[e] = su;
          }
          for (int64_t q2 = blo; q2 < bhi; ++q2) {
            double sv = 0.0;
            for (int32_t e = 0; e < kb; ++e) sv += tmp[e] * Vbb[(q2 - blo) * kb + e];
            A[r * n + q2] = sv;
          }
        }
      }
    }
  free(tmp); free(Ub); free(Vb); free(bo);
  hss_teardown(&s);
  return 0;
}

int oracle_hss_dense_ranked(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks,
                            const double* D, const double* U, const double* V,
                            const double* R, const double* W, const double* B, double* A) {
  if (p < 0 || p > 40 || (p > 0 && !ranks)) return -1;
  int32_t* r = node_ranks_of_levels(p, ranks, 0);
  int rc = r ? oracle_hss_dense_noderanked(n, p, c, r, D, U, V, R, W, B, A) : -1;
  free(r);
  return rc;
}

int oracle_hss_dense(int64_t n, int32_t p, const int64_t* c, int32_t k,
                     const double* D, const double* U, const double* V,
                     const double* R, const double* W, const double* B, double* A) {
  if (k < 0 || p < 0 || p > 40) return -1;
  int32_t* r = node_ranks_of_levels(p, NULL, k);
  int rc = r ? oracle_hss_dense_noderanked(n, p, c, r, D, U, V, R, W, B, A) : -1;
  free(r);
  return rc;
}

/* --------------------------------------------------- hss2hodlr (f3) -- */

/* node (l, i), l >= 1, of the uniform-rank level-major arrays */
static int64_t coef_index(int32_t l, int64_t i) { return ((int64_t)1 << l) - 2 + i; }

/* P:522 ("hss2hodlr ... by simply building explicit low-rank factorizations",
 * S:514-522): the level-l bases of eq. (3),
 *   U_i^(l) = blockdiag(U_{2i}^(l+1), U_{2i+1}^(l+1)) R_{U,i}^(l), V likewise with
 *   R_{V,i}^(l) = W, built level by level from the leaves (U^(p) = U, V^(p) = V);
 * then every sibling block A(I_a, I_b) = U_a^(l) S_ab V_b^(l)* is
 * the HODLR block U_l(I_a) V_l(I_b)^* with U_l(I_a) = U_a^(l) S_ab (S = B12
 * for a = 2q, B21 for a = 2q+1 of the parent q) and V_l(I_b) = V_b^(l).
 * Output: Uh, Vh level-major [p][n][k] (the HODLR layout with ranks k). Exact
 * (no truncation). Sums in natural order. */
int oracle_hss_to_hodlr(int64_t n, int32_t p, const int64_t* c, int32_t k,
                        const double* U, const double* V, const double* R, const double* W,
                        const double* B, double* Uh, double* Vh) {
  if (check_tree(n, p, c) || k < 0 || (p > 0 && (!Uh || !Vh))) return -1;
  if (p == 0 || k == 0) return 0;
  const size_t nk = (size_t)n * (size_t)k;
  double* Ucur = (double*)malloc(sizeof(double) * nk); /* U^(l): rows I_i^l hold U_i^(l) */
  double* Unext = (double*)malloc(sizeof(double) * nk);
  if (!Ucur || !Unext) { free(Ucur); free(Unext); return -1; }
  memcpy(Ucur, U, sizeof(double) * nk);
  memcpy(Vh + (size_t)(p - 1) * nk, V, sizeof(double) * nk); /* V_p = V^(p) */
  for (int32_t l = p; l >= 1; --l) {
    double* Ul = Uh + (size_t)(l - 1) * nk;
    double* Vl = Vh + (size_t)(l - 1) * nk;
    /* U_l(I_a) = U_a^(l) S_{a, sib a} */
    for (int64_t a = 0; a < ((int64_t)1 << l); ++a) {
      int64_t lo, hi;
      node_range(c, p, l, a, &lo, &hi);
      const double* S = B + ((((int64_t)1 << (l - 1)) - 1 + (a >> 1)) * 2 + (a & 1)) * k * k;
      for (int64_t r = lo; r < hi; ++r)
        for (int32_t e = 0; e < k; ++e) {
          double s = 0.0;
          for (int32_t f = 0; f < k; ++f) s += Ucur[r * k + f] * S[f * k + e];
          Ul[r * k + e] = s;
        }
    }
    if (l == 1) break;
    /* eq. (3): U^(l-1), V^(l-1) from the level-l bases and the translations of
     * the level-(l-1) nodes: rows of child ch of node i get U^(l) R_ch, V^(l) W_ch */
    for (int64_t i = 0; i < ((int64_t)1 << (l - 1)); ++i)
      for (int ch = 0; ch < 2; ++ch) {
        int64_t lo, hi;
        node_range(c, p, l, 2 * i + ch, &lo, &hi);
        const double* Rh = R + coef_index(l - 1, i) * 2 * k * k + ch * k * k;
        const double* Wh = W + coef_index(l - 1, i) * 2 * k * k + ch * k * k;
        for (int64_t r = lo; r < hi; ++r)
          for (int32_t e = 0; e < k; ++e) {
            double su = 0.0, sv = 0.0;
            for (int32_t f = 0; f < k; ++f) {
              su += Ucur[r * k + f] * Rh[f * k + e];
              sv += Vl[r * k + f] * Wh[f * k + e];
            }
            Unext[r * k + e] = su;
            Vh[(size_t)(l - 2) * nk + r * k + e] = sv;
          }
      }
    double* t = Ucur; Ucur = Unext; Unext = t;
  }
  free(Ucur); free(Unext);
  return 0;
}

/* ------------------------------------------------- norm estimate (f2) -- */
/* Power method on A A^* ("estimating ||A||_2 by means of the power
 * method on AA^*"; SPEC S:165-173 estimate_norm2): with v_0 = x0/||x0||,
 *   w_j = A^* v_{j-1},  eta_j = ||w_j||_2,  z_j = A w_j,  v_j = z_j/||z_j||_2,
 * j = 1..iters; returns eta_iters (0 for the zero operator). eta_j = ||A^* v||
 * for a unit v, so eta_j <= ||A||_2 (reading R-f2 in DESIGN.md). Norms are
 * sqrt of a sequential sum of squares in natural order. */
static double vec_norm2(int64_t n, const double* v) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += v[i] * v[i];
  return sqrt(s);
}

typedef int (*apply_fn)(const void* ctx, int trans, const double* x, double* y);

static int power_norm2(int64_t n, const double* x0, int32_t iters, apply_fn f, const void* ctx, double* est) {
  if (n < 1 || iters < 1 || !x0 || !est) return -1;
  double* v = (double*)malloc(sizeof(double) * (size_t)n);
  double* w = (double*)malloc(sizeof(double) * (size_t)n);
  if (!v || !w) { free(v); free(w); return -1; }
  double nv = vec_norm2(n, x0), eta = 0.0;
  int rc = 0;
  if (nv > 0.0) {
    for (int64_t i = 0; i < n; ++i) v[i] = x0[i] / nv;
    for (int32_t j = 1; j <= iters && rc == 0; ++j) {
      if ((rc = f(ctx, 1, v, w))) break;           /* w = A^* v */
      eta = vec_norm2(n, w);
      if (eta == 0.0) break;
      if ((rc = f(ctx, 0, w, v))) break;           /* z = A w (into v) */
      double nz = vec_norm2(n, v);
      for (int64_t i = 0; i < n; ++i) v[i] = v[i] / nz;
    }
  }
  free(v); free(w);
  *est = eta;
  return rc;
}

typedef struct {
  int64_t n; int32_t p; const int64_t* c; const int32_t* ranks; int32_t k;
  const double *D, *U, *V, *R, *W, *B;
} op_ctx;

static int hodlr_apply(const void* ctx, int trans, const double* x, double* y) {
  const op_ctx* o = (const op_ctx*)ctx;
  return hodlr_matvec_op(o->n, o->p, o->c, o->ranks, o->D, o->U, o->V, x, 1, y, trans);
}

static int hss_apply(const void* ctx, int trans, const double* x, double* y) {
  const op_ctx* o = (const op_ctx*)ctx;
  return hss_matvec_op(o->n, o->p, o->c, o->ranks, o->D, o->U, o->V, o->R, o->W, o->B, x, 1, y, trans);
}

int oracle_hodlr_norm2_est(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks,
                           const double* D, const double* U, const double* V,
                           const double* x0, int32_t iters, double* est) {
  op_ctx o = {n, p, c, ranks, 0, D, U, V, NULL, NULL, NULL};
  return power_norm2(n, x0, iters, hodlr_apply, &o, est);
}

int oracle_hss_norm2_est(int64_t n, int32_t p, const int64_t* c, int32_t k,
                         const double* D, const double* U, const double* V,
                         const double* R, const double* W, const double* B,
                         const double* x0, int32_t iters, double* est) {
  if (k < 0) return -1;
  int32_t* r = node_ranks_of_levels(p, NULL, k);
  if (!r) return -1;
  op_ctx o = {n, p, c, r, k, D, U, V, R, W, B};
  int rc = power_norm2(n, x0, iters, hss_apply, &o, est);
  free(r);
  return rc;
}

int oracle_dense_matvec(int64_t n, const double* A, const double* X, int32_t m, double* Y) {
  if (n < 0 || m < 1 || !A || !X || !Y) return -1;
  dense_mul(n, n, A, n, X, m, Y);
  return 0;
}

int oracle_laplacian_inverse_apply(int64_t n, const double* X, int32_t m, double* Y) {
  /* (tridiag(-1,2,-1))^{-1}_{ij} = min(i,j)(n+1-max(i,j))/(n+1), 1-based
   * (BASELINE.json config 5; eq. (8) P:1314-1322 is the same Laplacian up to
   * the factor -1/h^2). y_i = [(n+1-i) P_i + i Q_i]/(n+1),
   * P_i = sum_{j<=i} j x_j, Q_i = sum_{j>i} (n+1-j) x_j, in long double. */
  if (n < 1 || m < 1 || !X || !Y) return -1;
  long double* P = (long double*)malloc(sizeof(long double) * (size_t)n);
  long double* Q = (long double*)malloc(sizeof(long double) * (size_t)n);
  if (!P || !Q) { free(P); free(Q); return -1; }
  const long double np1 = (long double)(n + 1);
  for (int32_t q = 0; q < m; ++q) {
    long double acc = 0.0L;
    for (int64_t i = 1; i <= n; ++i) {
      acc += (long double)i * (long double)X[(i - 1) * m + q];
      P[i - 1] = acc;
    }
    acc = 0.0L;
    for (int64_t i = n; i >= 1; --i) {
      Q[i - 1] = acc; /* sum over j > i */
      acc += (np1 - (long double)i) * (long double)X[(i - 1) * m + q];
    }
    for (int64_t i = 1; i <= n; ++i)
      Y[(i - 1) * m + q] = (double)(((np1 - (long double)i) * P[i - 1] + (long double)i * Q[i - 1]) / np1);
  }
  free(P); free(Q);
  return 0;
}
