/*
 * hm.h — C-ABI of libhm: the B200 hot path of hm-toolbox (arXiv 1909.07909),
 * the fast hierarchical matrix–(multi)vector product Y = A·X in fp64 for
 *   - HODLR matrices (§4.1, Fig. 5 left P:666-678;
 *     format: Def. 2.2, class P:226-235), and
 *   - HSS matrices (§4.1, Fig. 5 right P:683-721; format: eq. (3)
 *     P:256-259, Def. 2.3, class P:332-344).
 * "P:n" = line n of /root/reference/PAPER.md. DESIGN.md §2 lists every
 * reading of an ambiguous passage (G1..G17) that these calls implement.
 *
 * Everything here is plain C: pointers, sizes, integers. No torch type, no
 * C++ type. All matrices are real fp64, ROW-MAJOR, contiguous.
 *
 * Memory and ownership
 *   - Generator arrays, X, Y and the workspace are DEVICE pointers on the
 *     calling thread's current CUDA device, owned by the caller. The library
 *     allocates no device memory, keeps no pointer after return, never
 *     synchronises the stream and never modifies an input (all inputs are
 *     const). Host-side state it does keep: a per-thread cache of the last 4
 *     general-tree (and per-node-rank HSS) plans, each with a pinned copy of the
 *     tables those calls copy into the workspace (pinned on first use, unpinned
 *     when the plan leaves the cache);
 *     the communicator of the multi-GPU calls owns an NCCL communicator, a
 *     stream and two events (hm_comm_init / hm_comm_destroy).
 *   - Exception: the *_hostio variants take X and Y as HOST pointers (pinned
 *     memory recommended; pageable works but serialises) and copy them
 *     through the workspace on `stream` — the end-to-end path.
 *   - `stream` is a cudaStream_t (CUstream) handle; NULL = legacy default.
 *     Work is enqueued asynchronously; results are valid once the stream has
 *     reached the point of the call.
 *   - Y is overwritten (Y = A X, not accumulated). X and Y must not overlap.
 *
 * Errors: every call returns an hm_status; on a negative status nothing was
 * enqueued (validation happens on the host before any launch) except for
 * HM_ERR_CUDA, which reports a launch failure. hm_last_error() returns a
 * thread-local, human-readable message for the last non-OK status. No call
 * aborts, exits or throws.
 *
 * Determinism: identical inputs on the same GPU give bitwise-identical Y
 * (no atomics, fixed reduction order) — SPEC S:343-344's deterministic mode.
 */
#ifndef HM_H
#define HM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HM_ABI_VERSION 2

typedef enum {
  HM_OK = 0,
  HM_ERR_INVALID_ARG = -1, /* inconsistent sizes, NULL/misaligned pointer, overlap */
  HM_ERR_UNSUPPORTED = -2, /* valid per the paper but not built (see each call)    */
  HM_ERR_WORKSPACE = -3,   /* workspace NULL or smaller than the query returned    */
  HM_ERR_CUDA = -4,        /* a CUDA launch / copy failed                          */
  HM_ERR_NCCL = -5         /* NCCL missing or failed (multi-GPU calls)             */
} hm_status;

/* Cluster tree (Def. 2.1). This build supports the balanced tree of
 * n = leaf * 2^levels, every level-l node I_i^l = [i*n/2^l, (i+1)*n/2^l)
 * (0-based), i.e. the default split of P:378-379 when n/leaf is a power of two.
 * levels = p = depth (root l = 0, leaves l = p); levels = 0 means A = D (one
 * dense block). General endpoint vectors (empty
 * leaves) use the *_general calls below. */
typedef struct {
  int64_t n;      /* matrix order, >= 1                                    */
  int32_t levels; /* p >= 0                                                */
  int32_t flags;  /* must be 0                                             */
  int64_t leaf;   /* leaf block size b >= 1, n == leaf << levels           */
} hm_tree;

/* ------------------------------------------------------------------ HODLR --
 * Generators (flat level-major layout; class fields of P:226-235):
 *   D  [2^p][b][b]   D_i = A(I_i^p, I_i^p), the dense leaves ("F").
 *   U  level-major:  level l = 1..p starts at offset n*sum_{l'<l} k_{l'} and
 *                    is [n][k_l]. Rows I_a^l of level l hold the left factor
 *                    of the sibling block (a, sib a):  A(I_a, I_b) =
 *                    U_l(I_a) V_l(I_b)^T for siblings a, b = a^1.
 *                    (U12 = U_l(I_2q), U21 = U_l(I_2q+1) of the parent q.)
 *   V  same shape as U; rows I_b of level l hold the right factor of block
 *                    (sib b, b). (V12 = V_l(I_2q+1), V21 = V_l(I_2q).)
 *   ranks [p] (host array): ranks[l-1] = k_l >= 0 (0 encodes the zero
 *                    block), each <= 64. Equal nonzero ranks run the
 *                    tuned kernels. Per-level ranks also run the
 *                    uniform-tree kernels when levels >= 3 and leaf is a
 *                    multiple of 64 (<= 1024): one V^T X pass per distinct
 *                    rank, one leaf pass with per-level segments; otherwise
 *                    the general-tree kernels (hodlr_matvec_general), with
 *                    the same workspace query either way (HM_WS_HOSTIO: the
 *                    uniform-tree case only).
 *   X  [n][nrhs], Y [n][nrhs]; nrhs >= 1.
 * Cost O(k n log n); bytes = 8(n b + 2 sum_l n k_l + 2 n nrhs). */

/* Workspace bytes for hodlr_matvec (flags = 0) or hodlr_matvec_hostio
 * (flags = HM_WS_HOSTIO). Returns HM_OK and writes *bytes. */
#define HM_WS_HOSTIO 1
hm_status hm_hodlr_workspace_bytes(const hm_tree* tree, const int32_t* ranks, int32_t nrhs,
                                   int32_t flags, size_t* bytes);

/* Y = A X for a HODLR matrix A, computed as Fig. 5 left prescribes
 * (y1+y2 / y3+y4 at every level) but level-parallel: all V_l^T X products
 * first, then each leaf's rows receive D_i X(I_i) + sum_l U_l t_{l,sib}. */
hm_status hodlr_matvec(const hm_tree* tree, const int32_t* ranks,
                       const double* D, const double* U, const double* V,
                       const double* X, int32_t nrhs, double* Y,
                       void* workspace, size_t workspace_bytes, void* stream);

/* Adjoint product Y = A^T X ("A^*" of P:404, the
 * Afunt handle of P:433-438; real data, so * is the transpose, reading G4).
 * Same arguments, layouts, workspace query (flags = 0), errors and
 * determinism as hodlr_matvec. A^T is HODLR on the same tree with the factor
 * roles exchanged, A^T(I_a, I_b) = V_l(I_a) U_l(I_b)^T, and leaf blocks D_i^T:
 * computed as U_l^T X contractions, then D_i^T X(I_i) + sum_l V_l(I_i) t_l. */
hm_status hodlr_matvec_t(const hm_tree* tree, const int32_t* ranks,
                         const double* D, const double* U, const double* V,
                         const double* X, int32_t nrhs, double* Y,
                         void* workspace, size_t workspace_bytes, void* stream);

/* Same, with X and Y in HOST memory (copied on `stream` through the
 * workspace; query with HM_WS_HOSTIO). */
hm_status hodlr_matvec_hostio(const hm_tree* tree, const int32_t* ranks,
                              const double* D, const double* U, const double* V,
                              const double* X_host, int32_t nrhs, double* Y_host,
                              void* workspace, size_t workspace_bytes, void* stream);

/* -------------------------------------------------------------------- HSS --
 * Generators (class fields of P:332-344; uniform rank k):
 *   D  [2^p][b][b]           leaf diagonal blocks D_i.
 *   U, V [n][k]              leaf bases U_i^(p), V_i^(p) stacked by leaf rows.
 *   R, W [2^p-2][2k][k]      translation operators of node (l,i), l = 1..p-1,
 *                            at index 2^l-2+i: R = R_{U,i}^(l) = [Rl; Rr],
 *                            W = R_{V,i}^(l) = [Wl; Wr] (eq. (3); "W_U" of
 *                            P:337 is R_V, reading G3). Rows 0..k-1 belong
 *                            to the left child. Unused (may be NULL) if p < 2.
 *   B  [2^p-1][2][k][k]      core blocks of node (l,q), l = 0..p-1, at index
 *                            2^l-1+q: [0] = B12 = S_{2q,2q+1}^(l+1),
 *                            [1] = B21 = S_{2q+1,2q}^(l+1).
 *   k in [0, 64]; k = 0 makes A block diagonal (G17). X, Y as for HODLR.
 * Cost O(k n). */
hm_status hm_hss_workspace_bytes(const hm_tree* tree, int32_t k, int32_t nrhs, int32_t flags,
                                 size_t* bytes);

/* Y = A X for an HSS matrix A: Step 1 (leaf V^T X, upsweep through W^T),
 * Step 2 (cores B, on every level l = 1..p — reading G1 of the garbled loop
 * bounds at P:695-706), Step 3 (downsweep through R), Step 4
 * (Y(I_i) = U_i y_i + D_i X(I_i), reading G2). */
hm_status hss_matvec(const hm_tree* tree, int32_t k,
                     const double* D, const double* U, const double* V,
                     const double* R, const double* W, const double* B,
                     const double* X, int32_t nrhs, double* Y,
                     void* workspace, size_t workspace_bytes, void* stream);

/* Adjoint product Y = A^T X. Same arguments, workspace
 * query, errors and determinism as hss_matvec. A^T is HSS on the same tree
 * with row bases V (translations W), column bases U (translations R), cores
 * S'_{2q,2q+1} = B21^T, S'_{2q+1,2q} = B12^T and leaf blocks D_i^T; the four
 * steps of Fig. 5 right run on those generators (no copy is made). */
hm_status hss_matvec_t(const hm_tree* tree, int32_t k,
                       const double* D, const double* U, const double* V,
                       const double* R, const double* W, const double* B,
                       const double* X, int32_t nrhs, double* Y,
                       void* workspace, size_t workspace_bytes, void* stream);

hm_status hss_matvec_hostio(const hm_tree* tree, int32_t k,
                            const double* D, const double* U, const double* V,
                            const double* R, const double* W, const double* B,
                            const double* X_host, int32_t nrhs, double* Y_host,
                            void* workspace, size_t workspace_bytes, void* stream);

/* -------------------------------- HSS with per-level ranks (§8(f) f4) --
 * the bases and translation operators need not have k columns on every
 * level, "as long as the dimensions are compatible". Level l = 1..p has rank
 * k_l = ranks[l-1] (0..64; 0 = no off-diagonal coupling through that level):
 *   U, V [n][k_p]              leaf bases.
 *   R, W                       node (l, i), l = 1..p-1: [2k_{l+1}][k_l] at offset
 *                              sum_{l'<l} 2^l' 2 k_{l'+1} k_l' + i 2 k_{l+1} k_l
 *                              (rows 0..k_{l+1}-1: the left child).
 *   B                          cores of the level-l siblings 2q, 2q+1, stored at
 *                              the parent (l-1, q): [2][k_l][k_l] at offset
 *                              sum_{l'<l} 2^(l'-1) 2 k_l'^2 + q 2 k_l^2 ([0] = B12).
 *   D, X, Y                    as for hss_matvec. op = 0: Y = A X; 1: A^T X.
 * Equal ranks are exactly the layout of hss_matvec and run its kernels.
 * Otherwise Steps 1 and 4 run the leaf kernels with k_p and the tree levels one
 * launch per level. Same errors / determinism as hss_matvec. */
hm_status hm_hss_ranked_workspace_bytes(const hm_tree* tree, const int32_t* ranks, int32_t nrhs, size_t* bytes);
hm_status hss_matvec_ranked(const hm_tree* tree, const int32_t* ranks, int32_t op,
                            const double* D, const double* U, const double* V,
                            const double* R, const double* W, const double* B,
                            const double* X, int32_t nrhs, double* Y,
                            void* workspace, size_t workspace_bytes, void* stream);

/* -------------------------------- HSS with per-node ranks (§8(f) f4) --
 * P:264 in full: every node may have its own rank. node_ranks (HOST array of
 * 2^(p+1) - 2 entries): node (l, i), l = 1..p, has rank k_h = node_ranks[h],
 * h = 2^l - 2 + i, 0..64. Layout (row-major, heap order):
 *   U, V   leaf after leaf: leaf i's b x k_(p,i) rows.
 *   R, W   node (l, i), l = 1..p-1: [k_(l+1,2i) + k_(l+1,2i+1)][k_(l,i)]
 *          (rows of the left child first), nodes in heap order.
 *   B      parent (l-1, q), l = 1..p, heap order from the root: B12
 *          [k_(l,2q)][k_(l,2q+1)] then B21 [k_(l,2q+1)][k_(l,2q)].
 *   D, X, Y, op as for hss_matvec_ranked. Ranks equal within each level are the
 * per-level layout (and run that path directly). Otherwise the generators are
 * zero-padded into the per-level layout with K_l = the level's largest rank
 * (in the workspace; exact, the padding is zero) and the per-level path runs:
 * one extra pass over the generators. The table of padded blocks is copied to
 * the workspace asynchronously from the cached plan's pinned copy (not
 * CUDA-graph capturable: the first call of a tree pins its table). */
hm_status hm_hss_noderanked_workspace_bytes(const hm_tree* tree, const int32_t* node_ranks, int32_t nrhs,
                                            size_t* bytes);
hm_status hss_matvec_noderanked(const hm_tree* tree, const int32_t* node_ranks, int32_t op,
                                const double* D, const double* U, const double* V,
                                const double* R, const double* W, const double* B,
                                const double* X, int32_t nrhs, double* Y,
                                void* workspace, size_t workspace_bytes, void* stream);

/* ----------------------------------- general cluster trees (§8(f) f4) --
 * The cluster tree of depth `levels` = p given by its leaf endpoint vector
 * c (Def. 2.1): c is a HOST array of 2^p int64 values,
 * nondecreasing, c[2^p - 1] = n; leaf i holds rows [c[i-1], c[i]) (c[-1] = 0)
 * and may be EMPTY (Fig. 4); the level-l node i is the union of
 * its 2^(p-l) leaves. D concatenates the |I_i| x |I_i| leaf blocks (row-major)
 * in leaf order. HODLR ranks may differ per level, 0..64 each; U, V
 * are level-major with level l at offset n * sum_{l' < l} k_l', [n][k_l]. HSS
 * takes one rank k (0..64) and the generator layout of hss_matvec.
 *   op = 0: Y = A X;  op = 1: Y = A^T X (adjoint, §8(f) f1).
 * Limits: largest leaf + sum of ranks <= 20480 (shared-memory staging of a
 * leaf), else HM_ERR_UNSUPPORTED. Errors as for the uniform calls; c not
 * nondecreasing or c[2^p-1] != n is HM_ERR_INVALID_ARG. The tables derived
 * from c are planned on the host (cached per thread for the last 4 trees, each
 * plan with a pinned copy of its tables) and copied into the workspace with
 * one asynchronous copy: the call does not synchronise the stream (a plan
 * leaving the cache waits for its last copy before unpinning), but it is not
 * CUDA-graph capturable (the first call of a tree pins its tables). Deterministic.
 * (hodlr_matvec / hodlr_matvec_t route per-level ranks on uniform trees
 * with fewer than 3 levels or leaves not a multiple of 64 here
 * automatically, with the same workspace query.) */
hm_status hm_hodlr_general_workspace_bytes(int64_t n, int32_t levels, const int64_t* c, const int32_t* ranks,
                                           int32_t nrhs, size_t* bytes);
hm_status hodlr_matvec_general(int64_t n, int32_t levels, const int64_t* c, const int32_t* ranks, int32_t op,
                               const double* D, const double* U, const double* V,
                               const double* X, int32_t nrhs, double* Y,
                               void* workspace, size_t workspace_bytes, void* stream);
hm_status hm_hss_general_workspace_bytes(int64_t n, int32_t levels, const int64_t* c, int32_t k, int32_t nrhs,
                                         size_t* bytes);
hm_status hss_matvec_general(int64_t n, int32_t levels, const int64_t* c, int32_t k, int32_t op,
                             const double* D, const double* U, const double* V,
                             const double* R, const double* W, const double* B,
                             const double* X, int32_t nrhs, double* Y,
                             void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------- norm estimate (§8(f) f2) --
 * ||A||_2 estimate by the power method on A A^* ("estimating ||A||_2
 * by means of the power method on AA^*", run before every recompression;
 * SPEC S:165-173 estimate_norm2):
 *   v = x0/||x0||;  iters times:  w = A^T v,  eta = ||w||_2,  z = A w,  v = z/||z||_2
 * and *est = the last eta. For a unit v, eta = ||A^T v|| <= ||A||_2, and eta
 * is nondecreasing in the iteration count. A zero x0 or zero operator gives 0.
 *   x0   [n] device vector (start vector; not modified)
 *   iters >= 1 (HM_ERR_INVALID_ARG otherwise)
 *   est  ONE double in device memory, written on `stream` (async)
 * Workspace: the *_norm2_workspace_bytes query (the nrhs = 1 matvec
 * workspace plus two n-vectors and the norm partials). Every product runs
 * through hodlr_matvec / hodlr_matvec_t (hss_*); norms are fixed-order
 * reductions, so the result is bitwise repeatable. Capturable in a CUDA graph
 * (no synchronisation, no allocation). */
hm_status hm_hodlr_norm2_workspace_bytes(const hm_tree* tree, const int32_t* ranks, size_t* bytes);
hm_status hodlr_norm2_est(const hm_tree* tree, const int32_t* ranks,
                          const double* D, const double* U, const double* V,
                          const double* x0, int32_t iters, double* est,
                          void* workspace, size_t workspace_bytes, void* stream);
hm_status hm_hss_norm2_workspace_bytes(const hm_tree* tree, int32_t k, size_t* bytes);
hm_status hss_norm2_est(const hm_tree* tree, int32_t k,
                        const double* D, const double* U, const double* V,
                        const double* R, const double* W, const double* B,
                        const double* x0, int32_t iters, double* est,
                        void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------- hss2hodlr (§8(f) f3) --
 * Exact conversion HSS -> HODLR ("by simply building explicit low-rank
 * factorizations"): the level-l bases of eq. (3)
 * are built from the leaves, U^(l-1) = blockdiag(U^(l) children) R,
 * V^(l-1) likewise with W, and every sibling block U_a^(l) S_ab V_b^(l)T
 * becomes the HODLR block U_l(I_a) V_l(I_b)^T with
 *   U_l(I_a) = U_a^(l) S_{a, sib a} (B12 for a = 2q, B21 for a = 2q+1),
 *   V_l(I_b) = V_b^(l).
 * Inputs: the HSS generators U, V [n][k], R, W, B as for hss_matvec.
 * Outputs: Uh, Vh [levels][n][k] device, the HODLR U, V of hodlr_matvec with
 * ranks[l-1] = k on every level; the HODLR leaf blocks are the HSS D
 * unchanged (reuse the same buffer). Uh, Vh must not overlap each other or
 * an input (HM_ERR_INVALID_ARG). levels = 0 or k = 0 writes nothing. No
 * workspace; O(k^2 n log n) flops, O(k n log n) bytes written; async on
 * `stream`; bitwise repeatable. */
hm_status hss_to_hodlr(const hm_tree* tree, int32_t k,
                       const double* U, const double* V, const double* R, const double* W, const double* B,
                       double* Uh, double* Vh, void* stream);

/* ---------------------------------------------------- multi-GPU (§8(e)) --
 * One process per GPU, P = 2^q ranks (1 <= P <= 2^levels). Rank r owns the
 * rows I_r = [r n/P, (r+1) n/P) — the level-q node (q, r) and its whole
 * subtree (Def. 2.1) — and these generators ("local" arrays):
 *   HODLR  D_local [2^(p-q)][b][b]; U_local, V_local level-major over ALL p
 *          levels with n/P rows each: level l at offset (n/P) sum_{l'<l} k_l',
 *          [n/P][k_l] = rows I_r of the global U_l, V_l. X_local, Y_local
 *          [n/P][nrhs] = rows I_r. One rank (uniform) for all levels.
 *   HSS    D_local, U_local, V_local [n/P][k] likewise; the subtree's W_sub,
 *          R_sub [2^(p-q)-2][2k][k] and B_sub [2^(p-q)-1][2][k][k] in heap
 *          order relative to node (q, r) (B_sub[0] = the cores of node (q,r));
 *          W_root, R_root [2k][k] = the translations of node (q, r) itself;
 *          W_top, R_top [2^q-2][2k][k] and B_top [2^q-1][2][k][k] = the global
 *          arrays' prefixes (levels < q), replicated on every rank.
 * The ONLY exchange is an allgather of small coefficient blocks per product:
 *   HODLR  rank r's partial t_l = V_l(I_r)^T X(I_r) for the top levels
 *          l = 1..q (q k nrhs doubles; config 5 at P = 8: 24 bytes). Each rank
 *          then sums, per top level, the partials of the ranks under the
 *          sibling of its ancestor (rank order) and adds U_l(I_r) t_l.
 *   HSS    x of node (q, r) (Step 1 up to the subtree root, k nrhs doubles);
 *          every rank runs the replicated top tree (levels 1..q), then its
 *          subtree's coupling / downsweep from y of node (q, r), and Step 4.
 * Results equal the single-GPU product up to the order of the top-level sums. */

/* ---- communicator: NCCL (loaded at run time from libnccl.so.2), one per
 * process, bound to the CUDA device current at hm_comm_init. Its allgather runs
 * on the communicator's own stream, ordered against the caller's stream with
 * events. Not thread-safe: one product at a time per communicator, issued in
 * the same order on every rank. */
typedef struct hm_comm_s hm_comm;
#define HM_COMM_ID_BYTES 128

/* Rank 0 creates the id and hands it to the other ranks out of band (the
 * Python binding broadcasts it through torch.distributed; examples/ uses a
 * pipe). HM_ERR_NCCL if NCCL cannot be loaded or fails. */
hm_status hm_comm_unique_id(void* id_out /* HM_COMM_ID_BYTES bytes */);
/* Collective over the nranks processes (blocks until all joined). nranks must
 * be a power of two (HM_ERR_UNSUPPORTED otherwise); the current CUDA device
 * must differ between the ranks (NCCL). *comm_out = NULL on failure. */
hm_status hm_comm_init(int32_t nranks, int32_t rank, const void* id, hm_comm** comm_out);
/* Waits for the communicator's stream, then frees it. NULL is a no-op. */
hm_status hm_comm_destroy(hm_comm* comm);
hm_status hm_comm_size(const hm_comm* comm, int32_t* nranks, int32_t* rank);
/* recv[P][count] <- every rank's send[count], rank order (the exchange
 * primitive of the products below), ordered after the work already on
 * `stream`; work enqueued on `stream` afterwards sees recv complete. In place
 * when send == recv + rank * count. */
hm_status hm_comm_allgather(hm_comm* comm, const double* send, int64_t count, double* recv, void* stream);

/* ---- the products, one call each (every rank calls with its local arrays).
 * The current device must be the communicator's. Per-level HODLR ranks are
 * not supported here (HM_ERR_UNSUPPORTED). Workspace: the query below (the
 * same on every rank). HM_ERR_NCCL if the exchange fails.
 * HODLR: the allgather runs while this rank computes its subtree's V^T X and
 * — when the extra Y read + write costs at most 3% of the bytes — its leaf
 * pass; the top-level terms are then added.
 * HSS: nothing local is independent of y of node (q, r) after Step 1, so the
 * allgather (k nrhs doubles per rank) is not overlapped. */
hm_status hm_hodlr_dist_workspace_bytes(const hm_tree* tree, const int32_t* ranks, int32_t nrhs, int32_t nranks,
                                        size_t* bytes);
hm_status hodlr_matvec_dist(hm_comm* comm, const hm_tree* tree, const int32_t* ranks, const double* D_local,
                            const double* U_local, const double* V_local, const double* X_local, int32_t nrhs,
                            double* Y_local, void* workspace, size_t workspace_bytes, void* stream);
hm_status hm_hss_dist_workspace_bytes(const hm_tree* tree, int32_t k, int32_t nrhs, int32_t nranks, size_t* bytes);
hm_status hss_matvec_dist(hm_comm* comm, const hm_tree* tree, int32_t k, const double* D_local,
                          const double* U_local, const double* V_local, const double* R_sub, const double* W_sub,
                          const double* B_sub, const double* R_root, const double* W_root, const double* R_top,
                          const double* W_top, const double* B_top, const double* X_local, int32_t nrhs,
                          double* Y_local, void* workspace, size_t workspace_bytes, void* stream);

/* ---- split-phase interface: the same products with the exchange done by the
 * caller (any transport; the tests use it to run every rank's kernels on one
 * GPU with the allgather replaced by a concatenation). The caller allgathers
 * `send_doubles` doubles per rank from `send` into `gathered` [P][send_doubles]
 * (rank order) between _begin and _end:
 *   HODLR  _begin (top partials into send); _local (the subtree's V^T X and,
 *          when hodlr_matvec_dist would overlap it, the leaf pass without the
 *          top levels — may run while the allgather is in flight); _end.
 *   HSS    _begin (send = x of node (q, r)); _end. */
typedef struct {
  int32_t nranks; /* P, a power of two <= 2^levels */
  int32_t rank;   /* 0 <= rank < P                  */
} hm_part;

hm_status hm_hodlr_dist_sizes(const hm_tree* tree, const int32_t* ranks, int32_t nrhs, const hm_part* part,
                              size_t* ws_bytes, int64_t* send_doubles);
hm_status hodlr_matvec_dist_begin(const hm_tree* tree, const int32_t* ranks, const hm_part* part,
                                  const double* V_local, const double* X_local, int32_t nrhs, double* send,
                                  void* workspace, size_t workspace_bytes, void* stream);
hm_status hodlr_matvec_dist_local(const hm_tree* tree, const int32_t* ranks, const hm_part* part,
                                  const double* D_local, const double* U_local, const double* V_local,
                                  const double* X_local, int32_t nrhs, double* Y_local, void* workspace,
                                  size_t workspace_bytes, void* stream);
hm_status hodlr_matvec_dist_end(const hm_tree* tree, const int32_t* ranks, const hm_part* part,
                                const double* D_local, const double* U_local, const double* X_local, int32_t nrhs,
                                const double* gathered, double* Y_local, void* workspace, size_t workspace_bytes,
                                void* stream);

hm_status hm_hss_dist_sizes(const hm_tree* tree, int32_t k, int32_t nrhs, const hm_part* part, size_t* ws_bytes,
                            int64_t* send_doubles);
hm_status hss_matvec_dist_begin(const hm_tree* tree, int32_t k, const hm_part* part, const double* V_local,
                                const double* W_sub, const double* W_root, const double* X_local, int32_t nrhs,
                                double* send, void* workspace, size_t workspace_bytes, void* stream);
hm_status hss_matvec_dist_end(const hm_tree* tree, int32_t k, const hm_part* part, const double* D_local,
                              const double* U_local, const double* R_sub, const double* B_sub,
                              const double* R_root, const double* W_top, const double* R_top, const double* B_top,
                              const double* X_local, int32_t nrhs, const double* gathered, double* Y_local,
                              void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------ misc -- */

/* Thread-local message describing the last non-OK status ("" if none). */
const char* hm_last_error(void);

/* HM_ABI_VERSION of the loaded library. */
int32_t hm_abi_version(void);

/* Number of kernel launches the last successful matvec call on this thread
 * enqueued (bench bookkeeping for "gpu_launches"). */
int32_t hm_last_launch_count(void);

/* Launch tracing (the measurement hook bench.py uses for per-kernel roofline
 * numbers). While enabled, every kernel launch of every matvec call is
 * bracketed by two CUDA events recorded on the launch's stream (no
 * synchronisation, ~1 us of host work per launch). hm_profile_collect waits
 * for the recorded events, writes up to `cap` records in launch order and
 * clears the trace. `call` numbers the matvec calls since the trace began.
 * `start_ms` places every record on one device timeline (it is measured from
 * the first record's start event, whatever stream either was recorded on), so
 * records of different streams — the distributed product's exchange on the
 * communicator's stream ("nccl_allgather") and the kernels on the caller's
 * stream — show whether they overlapped. */
typedef struct {
  char name[40];  /* kernel name, e.g. "leaf_apply", "vt_contract" */
  int32_t call;   /* index of the matvec call that launched it      */
  float ms;       /* device time between the bracketing events      */
  float start_ms; /* start event minus the trace's first start event */
} hm_launch_record;

hm_status hm_profile_enable(int32_t on);
hm_status hm_profile_collect(hm_launch_record* out, int32_t cap, int32_t* count);

#ifdef __cplusplus
}
#endif
#endif /* HM_H */
