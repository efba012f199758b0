/*
 * hm_oracle.h — CPU ORACLE for the HODLR / HSS matrix–(multi)vector product.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing on the product path (libhm, its kernels,
 * its Python binding) may include, link, load or call anything declared here.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs use it. It shares no code, header, table or helper
 * with paper_1909_07909_b200/csrc.
 *
 * Paper: hm-toolbox (arXiv 1909.07909), /root/reference/PAPER.md, cited "P:n"
 * by line. Every routine follows the paper's definitions and pseudocode in
 * their order and notation; see each function's comment.
 *
 * Conventions (DESIGN.md §3 "Readings"):
 *   - all matrices real fp64, row-major; "*" (conjugate transpose) reads as
 *     transpose (reading G4);
 *   - a cluster tree of depth p is given by its leaf endpoint vector
 *     c[0..2^p-1]: leaf i (0-based) holds rows [c[i-1], c[i]),
 *     c[-1] := 0; empty leaves allowed (Fig. 4). The level-l node i
 *     holds rows [c[i*2^(p-l) - 1], c[(i+1)*2^(p-l) - 1]) (Def. 2.1);
 *   - levels l = 0 (root) .. p (leaves); nodes 0-based; sibling pairs
 *     (2q, 2q+1) under parent q.
 *
 * Generator layouts (the same flat level-major layout the C-ABI uses; the
 * oracle re-derives its own indexing, it does not share the product's):
 *   D : leaf blocks D_i = A(I_i^p, I_i^p) concatenated, block i is
 *       |I_i| x |I_i| row-major (uniform tree: [2^p][b][b]).
 *   HODLR U, V : level-major; level l (1..p) at offset n*sum_{l'<l} k_{l'},
 *       shape [n][k_l]. Rows I_a of level l hold U-factor of block (a, sib a)
 *       and V-factor of block (sib a, a):  A(I_a, I_b) = U_l(I_a) V_l(I_b)^T
 *       for siblings a, b (Def. 2.2; class P:226-235).
 *   HSS U, V : [n][k] leaf bases U_i^(p), V_i^(p) stacked by leaf rows.
 *   HSS R, W : [2^p-2][2k][k]; node (l,i), l = 1..p-1, at index 2^l-2+i;
 *       rows 0..k-1 = Rl (left child), k..2k-1 = Rr (eq. (3)
 *       P:256-259; W is the column operator R_V, reading G3).
 *   HSS B : [2^p-1][2][k][k]; node (l,q), l = 0..p-1, at index 2^l-1+q;
 *       [0] = B12 = S_{2q,2q+1}^{(l+1)}, [1] = B21 = S_{2q+1,2q}^{(l+1)}.
 *   X, Y : [n][m] row-major.
 *
 * Return value: 0 on success, negative on invalid arguments.
 */
#ifndef HM_ORACLE_H
#define HM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Default cluster split: {1..ceil(n/2)} u {ceil(n/2)+1..n},
 * recursively until every set has cardinality <= nmin. Writes the depth to
 * *p_out and, if c_out != NULL, the 2^p leaf endpoints (capacity cap). */
int oracle_default_cluster(int64_t n, int64_t nmin, int32_t* p_out, int64_t* c_out, int64_t cap);

/* HODLR_matvec, Fig. 5 left, as a literal recursion. */
int oracle_hodlr_matvec(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks,
                        const double* D, const double* U, const double* V,
                        const double* X, int32_t m, double* Y);

/* Same recursion, evaluated only for the rows of the listed leaves.
 * Dsel holds the diagonal blocks of exactly those leaves, in list order.
 * Yout is [sum |I_leaf|][m], leaves in list order. Same arithmetic, in the
 * same order, as oracle_hodlr_matvec for those rows. */
int oracle_hodlr_matvec_leaves(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks,
                               const double* Dsel, const double* U, const double* V,
                               const double* X, int32_t m,
                               const int64_t* leaves, int64_t nleaves, double* Yout);

/* HSS_matvec, Fig. 5 right, four steps, with readings G1/G2. */
int oracle_hss_matvec(int64_t n, int32_t p, const int64_t* c, int32_t k,
                      const double* D, const double* U, const double* V,
                      const double* R, const double* W, const double* B,
                      const double* X, int32_t m, double* Y);

/* Same four steps; Steps 1 (V^T x part) and 2 in full, Steps 2'/3 (coupling,
 * downsweep) only along the root-to-leaf paths of the listed leaves, Step 4
 * only for those leaves. Dsel / Yout as for oracle_hodlr_matvec_leaves. */
int oracle_hss_matvec_leaves(int64_t n, int32_t p, const int64_t* c, int32_t k,
                             const double* Dsel, const double* U, const double* V,
                             const double* R, const double* W, const double* B,
                             const double* X, int32_t m,
                             const int64_t* leaves, int64_t nleaves, double* Yout);

/* Adjoint products Y = A^* X (reading G4: real, so A^T X) — SURVEY §8(f) f1.
 * A^* of a HODLR / HSS matrix has the same format on the same tree with the
 * generators' roles exchanged (U <-> V, R <-> W, cores transposed and
 * swapped, D_i transposed); each routine runs the same pseudocode (Fig. 5)
 * on those generators. Arguments as for the forward products. */
int oracle_hodlr_matvec_t(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks,
                          const double* D, const double* U, const double* V,
                          const double* X, int32_t m, double* Y);
int oracle_hodlr_matvec_t_leaves(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks,
                                 const double* Dsel, const double* U, const double* V,
                                 const double* X, int32_t m,
                                 const int64_t* leaves, int64_t nleaves, double* Yout);
int oracle_hss_matvec_t(int64_t n, int32_t p, const int64_t* c, int32_t k,
                        const double* D, const double* U, const double* V,
                        const double* R, const double* W, const double* B,
                        const double* X, int32_t m, double* Y);
int oracle_hss_matvec_t_leaves(int64_t n, int32_t p, const int64_t* c, int32_t k,
                               const double* Dsel, const double* U, const double* V,
                               const double* R, const double* W, const double* B,
                               const double* X, int32_t m,
                               const int64_t* leaves, int64_t nleaves, double* Yout);

/* ||A||_2 estimate by the power method on A A^* (SURVEY §8(f) f2):
 * v_0 = x0/||x0||; w = A^* v, eta = ||w||, z = A w, v = z/||z||, `iters`
 * times; *est = the last eta (<= ||A||_2; 0 for the zero operator). x0 [n]. */
int oracle_hodlr_norm2_est(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks,
                           const double* D, const double* U, const double* V,
                           const double* x0, int32_t iters, double* est);
int oracle_hss_norm2_est(int64_t n, int32_t p, const int64_t* c, int32_t k,
                         const double* D, const double* U, const double* V,
                         const double* R, const double* W, const double* B,
                         const double* x0, int32_t iters, double* est);

/* hss2hodlr: exact HODLR factors of an HSS matrix.
 * Uh, Vh: level-major [p][n][k] (HODLR layout, every rank k); the HODLR leaf
 * blocks are the HSS D unchanged. U_l(I_a) = U_a^(l) S_{a,sib a},
 * V_l(I_b) = V_b^(l), bases by eq. (3). */
int oracle_hss_to_hodlr(int64_t n, int32_t p, const int64_t* c, int32_t k,
                        const double* U, const double* V, const double* R, const double* W,
                        const double* B, double* Uh, double* Vh);

/* Dense matrix represented by the generators (n x n, row-major), by the
 * definitions: HODLR Def. 2.2; HSS off-diagonal blocks
 * U_i^(l) S_ij^(l) V_j^(l)T with bases rebuilt by eq. (3). */
int oracle_hodlr_dense(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks,
                       const double* D, const double* U, const double* V, double* A);
int oracle_hss_dense(int64_t n, int32_t p, const int64_t* c, int32_t k,
                     const double* D, const double* U, const double* V,
                     const double* R, const double* W, const double* B, double* A);

/* Per-level HSS ranks: k_l = ranks[l-1] on the nodes of level l = 1..p.
 * U, V [n][k_p]; R, W node (l,i) [2k_{l+1}][k_l] at offset
 * sum_{l'<l} 2^l' 2 k_{l'+1} k_l' + i 2 k_{l+1} k_l; B for the level-l siblings of
 * parent (l-1, q) [2][k_l][k_l] at sum_{l'<l} 2^(l'-1) 2 k_l'^2 + q 2 k_l^2. Equal
 * ranks give the uniform layout above (and the same result, bit for bit). */
int oracle_hss_matvec_ranked(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks,
                             const double* D, const double* U, const double* V,
                             const double* R, const double* W, const double* B,
                             const double* X, int32_t m, double* Y);
int oracle_hss_matvec_ranked_t(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks,
                               const double* D, const double* U, const double* V,
                               const double* R, const double* W, const double* B,
                               const double* X, int32_t m, double* Y);
int oracle_hss_dense_ranked(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks,
                            const double* D, const double* U, const double* V,
                            const double* R, const double* W, const double* B, double* A);

/* Per-node HSS ranks ("k columns for every level and node ... not
 * necessary"): node (l, i), l = 1..p, has rank node_ranks[2^l - 2 + i]. U, V:
 * leaf after leaf, |I_i| x k rows; R, W of node h (l = 1..p-1), heap order:
 * [k_{2i} + k_{2i+1}][k_h]; cores of parent (l-1, q), heap order from the
 * root: B12 [k_{2q}][k_{2q+1}] then B21 [k_{2q+1}][k_{2q}]. */
int oracle_hss_matvec_noderanked(int64_t n, int32_t p, const int64_t* c, const int32_t* node_ranks,
                                 const double* D, const double* U, const double* V,
                                 const double* R, const double* W, const double* B,
                                 const double* X, int32_t m, double* Y);
int oracle_hss_matvec_noderanked_t(int64_t n, int32_t p, const int64_t* c, const int32_t* node_ranks,
                                   const double* D, const double* U, const double* V,
                                   const double* R, const double* W, const double* B,
                                   const double* X, int32_t m, double* Y);
int oracle_hss_dense_noderanked(int64_t n, int32_t p, const int64_t* c, const int32_t* node_ranks,
                                const double* D, const double* U, const double* V,
                                const double* R, const double* W, const double* B, double* A);

/* Plain dense product Y = A X (n x n times n x m), sums in natural order. */
int oracle_dense_matvec(int64_t n, const double* A, const double* X, int32_t m, double* Y);

/* Inverse of tridiag(-1,2,-1) applied to X (BASELINE config 5):
 * A_ij = min(i,j)(n+1-max(i,j))/(n+1), 1-based, so
 * y_i = [(n+1-i) sum_{j<=i} j x_j + i sum_{j>i} (n+1-j) x_j] / (n+1).
 * Two prefix sums in long double, O(n m). Independent of any tree. */
int oracle_laplacian_inverse_apply(int64_t n, const double* X, int32_t m, double* Y);

/* Number of threads the OpenMP parts use (1 if built without OpenMP). */
int oracle_num_threads(void);
void oracle_set_num_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
