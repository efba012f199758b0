"""Pins for the CPU oracle (oracle/hm_oracle.c) — things other than the oracle itself.

Every check here compares the oracle with something the paper or mathematics
fixes: the paper's printed examples (tests/golden, cited), dense brute force
assembled in numpy directly from the definitions (Def. 2.2; eq. (3)
P:256-259), closed forms (inverse 1D Laplacian, BASELINE config 5), exact
structured cases ('eye', 'zeros', 'ones'), invariants (linearity,
column independence, symmetry), and thread-count independence.
"""
import os
import subprocess
import sys
from fractions import Fraction

import numpy as np
import pytest
import scipy.linalg

import oracle
import hm_inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------- numpy brute force (tests) --

def tree_sets(c, p, l):
    """Row ranges [lo, hi) of level l (Def. 2.1), from leaf endpoints c."""
    span = 1 << (p - l)
    out = []
    for i in range(1 << l):
        lo = 0 if i == 0 else int(c[i * span - 1])
        out.append((lo, int(c[(i + 1) * span - 1])))
    return out


def dense_hodlr_np(n, p, ranks, D, U, V, c):
    """A_rep from Def. 2.2: D_i on the diagonal, U_l(I_a) V_l(I_b)^T on sibling blocks."""
    A = np.zeros((n, n))
    off = 0
    for (lo, hi) in tree_sets(c, p, p):
        s = hi - lo
        A[lo:hi, lo:hi] = D[off: off + s * s].reshape(s, s)
        off += s * s
    uoff = 0
    for l in range(1, p + 1):
        k = ranks[l - 1]
        Ul = U[uoff: uoff + n * k].reshape(n, k)
        Vl = V[uoff: uoff + n * k].reshape(n, k)
        sets = tree_sets(c, p, l)
        for a in range(1 << l):
            (alo, ahi), (blo, bhi) = sets[a], sets[a ^ 1]
            A[alo:ahi, blo:bhi] = Ul[alo:ahi] @ Vl[blo:bhi].T
        uoff += n * k
    return A


def dense_hss_np(n, p, k, D, U, V, R, W, B, c):
    """A_rep from P:250-259: off-diagonal sibling blocks U_a^(l) S_ab V_b^(l)T with
    U^(l) = blockdiag(U^(l+1) children) R_U (eq. (3)), V likewise with R_V = W."""
    A = np.zeros((n, n))
    off = 0
    for (lo, hi) in tree_sets(c, p, p):
        s = hi - lo
        A[lo:hi, lo:hi] = D[off: off + s * s].reshape(s, s)
        off += s * s
    if p == 0 or k == 0:
        return A
    R = R.reshape(-1, 2 * k, k)
    W = W.reshape(-1, 2 * k, k)
    B = B.reshape(-1, 2, k, k)
    Ub = {p: [U.reshape(n, k)[lo:hi] for (lo, hi) in tree_sets(c, p, p)]}
    Vb = {p: [V.reshape(n, k)[lo:hi] for (lo, hi) in tree_sets(c, p, p)]}
    for l in range(p - 1, 0, -1):
        Ub[l], Vb[l] = [], []
        for i in range(1 << l):
            node = (1 << l) - 2 + i
            bdU = scipy.linalg.block_diag(Ub[l + 1][2 * i], Ub[l + 1][2 * i + 1])
            bdV = scipy.linalg.block_diag(Vb[l + 1][2 * i], Vb[l + 1][2 * i + 1])
            Ub[l].append(bdU @ R[node])
            Vb[l].append(bdV @ W[node])
    for l in range(1, p + 1):
        sets = tree_sets(c, p, l)
        for q in range(1 << (l - 1)):
            node = (1 << (l - 1)) - 1 + q
            a, b = 2 * q, 2 * q + 1
            A[sets[a][0]:sets[a][1], sets[b][0]:sets[b][1]] = Ub[l][a] @ B[node, 0] @ Vb[l][b].T
            A[sets[b][0]:sets[b][1], sets[a][0]:sets[a][1]] = Ub[l][b] @ B[node, 1] @ Vb[l][a].T
    return A


def relerr(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def random_hodlr_general(c, p, ranks, rng):
    n = int(c[-1])
    sizes = np.diff(np.concatenate([[0], c]))
    D = rng.standard_normal(int((sizes ** 2).sum()))
    U = rng.standard_normal(n * int(sum(ranks)))
    V = rng.standard_normal(n * int(sum(ranks)))
    return D, U, V


def random_hss_general(c, p, k, rng, orth=True):
    n = int(c[-1])
    sizes = np.diff(np.concatenate([[0], c]))
    D = rng.standard_normal(int((sizes ** 2).sum()))
    U = rng.standard_normal((n, k))
    V = rng.standard_normal((n, k))
    nt, nb = max((1 << p) - 2, 0), (1 << p) - 1
    R = rng.standard_normal((nt, 2 * k, k))
    W = rng.standard_normal((nt, 2 * k, k))
    B = rng.standard_normal((nb, 2, k, k))
    if orth:
        R = np.linalg.qr(R)[0] if nt else R
        W = np.linalg.qr(W)[0] if nt else W
    return D, U.ravel(), V.ravel(), R.ravel(), W.ravel(), B.ravel()


# ---------------------------------------------------------------- trees --

def _read_sets(path):
    rows, c = {}, None
    for line in open(path):
        if line.startswith("#") or not line.strip():
            continue
        key, val = line.split(":", 1)
        if key == "c":
            c = [int(v) for v in val.split()]
            continue
        sets = []
        for part in val.split("|"):
            part = part.strip()
            sets.append([] if part == "-" else [int(v) for v in part.split()])
        rows[int(key)] = sets
    return c, rows


def _sets_1based(c, p, l):
    return [list(range(lo + 1, hi + 1)) for (lo, hi) in tree_sets(c, p, l)]


def test_default_cluster_matches_fig1():
    _, gold = _read_sets(os.path.join(GOLD, "fig1_cluster_tree.txt"))
    p, c = oracle.default_cluster(8, 1)
    assert p == 3
    for l, sets in gold.items():
        assert _sets_1based(c, p, l) == sets


def test_endpoint_vector_matches_fig4():
    cg, gold = _read_sets(os.path.join(GOLD, "fig4_cluster_c.txt"))
    for l, sets in gold.items():
        assert _sets_1based(np.array(cg), 2, l) == sets


@pytest.mark.parametrize("n,nmin,p,c", [(1000, 256, 2, [250, 500, 750, 1000]), (5, 8, 0, [5]),
                                        (3, 1, 2, [1, 2, 3, 3]), (1024, 64, 4, [64 * (i + 1) for i in range(16)])])
def test_default_cluster_ceil_split(n, nmin, p, c):
    """first child {1..ceil(n/2)}; stop at n_min (SPEC examples S:41-43)."""
    pp, cc = oracle.default_cluster(n, nmin)
    assert pp == p and list(cc) == c


# ------------------------------------------------------- HODLR vs brute force --

@pytest.mark.parametrize("c,p,ranks,m", [
    ([32 * (i + 1) for i in range(16)], 4, [3, 5, 2, 4], 3),
    ([2, 4, 8, 8], 2, [1, 2], 2),                     # Fig. 4 tree, empty leaf
    ([5, 9, 9, 20, 21, 30, 33, 40], 3, [2, 0, 3], 1),  # ragged leaves, a rank-0 level
    ([7], 0, [], 4),                                   # depth-0 tree: Y = D X
])
def test_hodlr_oracle_vs_dense_definition(c, p, ranks, m):
    rng = np.random.default_rng(1)
    c = np.array(c)
    n = int(c[-1])
    D, U, V = random_hodlr_general(c, p, ranks, rng)
    X = rng.standard_normal((n, m))
    A = dense_hodlr_np(n, p, ranks, D, U, V, c)
    Y = oracle.hodlr_matvec(n, p, ranks, D, U, V, X, c=c)
    assert relerr(Y, A @ X) < 1e-14
    # the oracle's own densifier follows the same definition
    assert relerr(oracle.hodlr_dense(n, p, ranks, D, U, V, c=c), A) < 1e-15
    assert relerr(oracle.dense_matvec(A, X), A @ X) < 1e-14


def test_hodlr_oracle_config1_vs_dense():
    cfg = hm_inputs.CONFIGS[1]
    h = hm_inputs.hodlr_random(cfg.n, cfg.levels, [cfg.k] * cfg.levels, cid=1)
    X = hm_inputs.rhs(cfg.n, 1, cid=1)
    c = np.arange(1, 17) * 64
    A = dense_hodlr_np(cfg.n, cfg.levels, h.ranks, h.D, h.U, h.V, c)
    Y = oracle.hodlr_matvec(cfg.n, cfg.levels, h.ranks, h.D, h.U, h.V, X)
    assert relerr(Y, A @ X) < 1e-14


@pytest.mark.parametrize("level", [1, 2, 3, 4])
def test_hodlr_level_isolation(level):
    """G14: D = 0 and one level non-zero; the product is that level's sibling-swapped
    block matrix alone (so a level-local error cannot hide inside ||Y||)."""
    rng = np.random.default_rng(level)
    n, p, ranks = 256, 4, [2, 3, 4, 5]
    c = np.arange(1, 17) * 16
    D = np.zeros(16 * 16 * 16)
    U = rng.standard_normal(n * sum(ranks))
    V = rng.standard_normal(n * sum(ranks))
    off = 0
    for l in range(1, p + 1):
        if l != level:
            U[off: off + n * ranks[l - 1]] = 0
        off += n * ranks[l - 1]
    X = rng.standard_normal((n, 2))
    A = dense_hodlr_np(n, p, ranks, D, U, V, c)
    assert np.count_nonzero(A) > 0
    assert relerr(oracle.hodlr_matvec(n, p, ranks, D, U, V, X), A @ X) < 1e-14


# ---------------------------------------------------------- HSS vs brute force --

@pytest.mark.parametrize("c,p,k,m", [
    ([16 * (i + 1) for i in range(16)], 4, 3, 2),
    ([64 * (i + 1) for i in range(16)], 4, 8, 1),
    ([2, 4, 8, 8], 2, 1, 2),                       # Fig. 4 tree, empty leaf
    ([10, 20], 1, 4, 3),                           # p = 1: no translation operators
    ([12], 0, 2, 2),                               # depth 0: Y = D X
    ([8 * (i + 1) for i in range(8)], 3, 0, 2),    # k = 0: block diagonal (G17)
])
def test_hss_oracle_vs_dense_definition(c, p, k, m):
    rng = np.random.default_rng(7)
    c = np.array(c)
    n = int(c[-1])
    D, U, V, R, W, B = random_hss_general(c, p, k, rng)
    X = rng.standard_normal((n, m))
    A = dense_hss_np(n, p, k, D, U, V, R, W, B, c)
    Y = oracle.hss_matvec(n, p, k, D, U, V, R, W, B, X, c=c)
    assert relerr(Y, A @ X) < 1e-14
    assert relerr(oracle.hss_dense(n, p, k, D, U, V, R, W, B, c=c), A) < 1e-14


def test_hss_oracle_config2_vs_dense():
    cfg = hm_inputs.CONFIGS[2]
    s = hm_inputs.hss_random(cfg.n, cfg.levels, cfg.k, cid=2)
    X = hm_inputs.rhs(cfg.n, 16, cid=2)
    c = np.arange(1, 65) * 64
    A = dense_hss_np(cfg.n, cfg.levels, cfg.k, s.D, s.U, s.V, s.R, s.W, s.B, c)
    Y = oracle.hss_matvec(cfg.n, cfg.levels, cfg.k, s.D, s.U, s.V, s.R, s.W, s.B, X)
    assert relerr(Y, A @ X) < 1e-14


def test_hss_literal_coupling_range_is_wrong():
    """Reading G1: Fig. 5 right's Step-2 loop literally stops at l = p-1; then the
    leaf-sibling cores S^(p) (Def. 2.3 / eq. at) would never be applied. With
    the leaf-level cores zeroed, the oracle must equal the dense matrix WITHOUT the
    level-p blocks — i.e. the oracle does apply level p when they are present."""
    rng = np.random.default_rng(3)
    n, p, k = 128, 3, 2
    c = np.arange(1, 9) * 16
    D, U, V, R, W, B = random_hss_general(c, p, k, rng)
    B = B.reshape(-1, 2, k, k)
    X = rng.standard_normal((n, 1))
    full = oracle.hss_matvec(n, p, k, D, U, V, R, W, B.ravel(), X)
    Bz = B.copy()
    Bz[(1 << (p - 1)) - 1:] = 0  # parents at level p-1 hold the leaf-level cores
    trunc = oracle.hss_matvec(n, p, k, D, U, V, R, W, Bz.ravel(), X)
    A_full = dense_hss_np(n, p, k, D, U, V, R, W, B.ravel(), c)
    assert relerr(full, A_full @ X) < 1e-14
    assert relerr(trunc, A_full @ X) > 1e-3


def test_hss_to_hodlr_cross_check():
    """P:522 / S:514-522: explicit factors of every off-diagonal block from the
    nested form (eq. (3)) give an exact HODLR representation; the two oracles
    must agree to rounding."""
    rng = np.random.default_rng(11)
    n, p, k, m = 512, 4, 4, 3
    c = np.arange(1, 17) * 32
    D, U, V, R, W, B = random_hss_general(c, p, k, rng)
    Rr, Wr, Br = R.reshape(-1, 2 * k, k), W.reshape(-1, 2 * k, k), B.reshape(-1, 2, k, k)
    Ub = {p: U.reshape(n, k).copy()}
    Vb = {p: V.reshape(n, k).copy()}
    for l in range(p - 1, 0, -1):
        Ub[l] = np.empty((n, k)); Vb[l] = np.empty((n, k))
        for i in range(1 << l):
            node = (1 << l) - 2 + i
            for ch in range(2):
                lo, hi = tree_sets(c, p, l + 1)[2 * i + ch]
                Ub[l][lo:hi] = Ub[l + 1][lo:hi] @ Rr[node, ch * k:(ch + 1) * k]
                Vb[l][lo:hi] = Vb[l + 1][lo:hi] @ Wr[node, ch * k:(ch + 1) * k]
    # HODLR level l: U_l(I_a) = U^(l)_a S_{a,b}, V_l(I_b) = V^(l)_b
    Uh, Vh = [], []
    for l in range(1, p + 1):
        Ul = np.empty((n, k))
        sets = tree_sets(c, p, l)
        for a in range(1 << l):
            lo, hi = sets[a]
            node = (1 << (l - 1)) - 1 + (a >> 1)
            Ul[lo:hi] = Ub[l][lo:hi] @ Br[node, a & 1]
        Uh.append(Ul.ravel()); Vh.append(Vb[l].ravel())
    X = rng.standard_normal((n, m))
    Yh = oracle.hodlr_matvec(n, p, [k] * p, D, np.concatenate(Uh), np.concatenate(Vh), X)
    Ys = oracle.hss_matvec(n, p, k, D, U, V, R, W, B, X)
    assert relerr(Ys, Yh) < 1e-14


# ------------------------------------------------------------ closed forms --

def test_laplacian_closed_form_golden():
    lines = [l for l in open(os.path.join(GOLD, "inv_laplacian_n8.txt")) if not l.startswith("#")]
    for xl, yl in zip(lines[0::2], lines[1::2]):
        x = np.array([float(v) for v in xl.split(":")[1].split()])
        y = [Fraction(v) for v in yl.split(":")[1].split()]
        yo = oracle.laplacian_inverse_apply(x)[:, 0]
        assert np.array_equal(yo, np.array([float(v) for v in y]))
        # and through the HODLR form of Fig. 1's tree (n = 8, n_min = 1, p = 3, k = 1)
        h = hm_inputs.hodlr_inverse_laplacian(8, 3)
        yh = oracle.hodlr_matvec(8, 3, h.ranks, h.D, h.U, h.V, x)[:, 0]
        assert np.max(np.abs(yh - np.array([float(v) for v in y]))) < 1e-13 * max(1, np.max(np.abs(yo)))


def _tridiag_residual(Y, X):
    """G12 / P:1248 normalisation: ||T Y - X|| / (||T||_2 ||Y|| + ||X||), T = tridiag(-1,2,-1)."""
    TY = 2 * Y
    TY[1:] -= Y[:-1]
    TY[:-1] -= Y[1:]
    n = Y.shape[0]
    normT = 2 + 2 * np.cos(np.pi / (n + 1))
    return np.linalg.norm(TY - X) / (normT * np.linalg.norm(Y) + np.linalg.norm(X))


@pytest.mark.parametrize("n,p", [(1 << 12, 4), (1 << 14, 6)])
def test_laplacian_oracle_vs_banded_solve(n, p):
    rng = np.random.default_rng(n)
    X = rng.standard_normal((n, 2))
    ab = np.zeros((3, n)); ab[0, 1:] = -1; ab[1] = 2; ab[2, :-1] = -1
    Ysolve = scipy.linalg.solve_banded((1, 1), ab, X)
    Y = oracle.laplacian_inverse_apply(X)
    # a backward-stable banded solve is only accurate to ~cond(T) eps, cond(T) ~ 4(n+1)^2/pi^2
    kappa = 4 * (n + 1) ** 2 / np.pi ** 2
    assert relerr(Y, Ysolve) < 10 * kappa * np.finfo(float).eps
    assert _tridiag_residual(Y, X) < 1e-15


def test_laplacian_oracle_vs_exact_rationals():
    """Exact A x in rational arithmetic (x's doubles taken exactly): the long-double
    prefix-sum oracle must be correctly rounded up to a few ulps."""
    n = 2048
    X = np.random.default_rng(2).standard_normal(n)
    xf = [Fraction(float(v)) for v in X]
    P, acc = [], Fraction(0)
    for i in range(1, n + 1):
        acc += i * xf[i - 1]
        P.append(acc)
    Q, acc = [Fraction(0)] * n, Fraction(0)
    for i in range(n, 0, -1):
        Q[i - 1] = acc
        acc += (n + 1 - i) * xf[i - 1]
    exact = np.array([float(((n + 1 - i) * P[i - 1] + i * Q[i - 1]) / (n + 1)) for i in range(1, n + 1)])
    Y = oracle.laplacian_inverse_apply(X)[:, 0]
    assert relerr(Y, exact) < 1e-15


@pytest.mark.parametrize("n,p", [(1 << 12, 4), (1 << 16, 8)])
def test_hodlr_inverse_laplacian_closed_form(n, p):
    h = hm_inputs.hodlr_inverse_laplacian(n, p)
    X = hm_inputs.rhs(n, 1, cid=5)
    Y = oracle.hodlr_matvec(n, p, h.ranks, h.D, h.U, h.V, X)
    assert relerr(Y, oracle.laplacian_inverse_apply(X)) < 1e-13
    assert _tridiag_residual(Y, X) < 1e-14


@pytest.mark.parametrize("n,p", [(1 << 10, 4), (1 << 14, 7)])
def test_hss_inverse_laplacian_closed_form(n, p):
    s = hm_inputs.hss_inverse_laplacian(n, p)
    X = hm_inputs.rhs(n, 2, cid=5)
    Y = oracle.hss_matvec(n, p, s.k, s.D, s.U, s.V, s.R, s.W, s.B, X)
    assert relerr(Y, oracle.laplacian_inverse_apply(X)) < 1e-13
    assert _tridiag_residual(Y, X) < 1e-14


# ---------------------------------------------------- exact structured cases --

def test_identity_zeros_ones_hodlr():
    n, p = 256, 3
    b = n >> p
    rng = np.random.default_rng(0)
    X = rng.standard_normal((n, 3))
    eye = np.tile(np.eye(b).ravel(), 1 << p)
    # 'eye': rank 0 on every level, D_i = I  ->  Y == X exactly
    Y = oracle.hodlr_matvec(n, p, [0] * p, eye, np.zeros(0), np.zeros(0), X)
    assert np.array_equal(Y, X)
    # 'zeros': Y == 0 exactly
    Y = oracle.hodlr_matvec(n, p, [0] * p, np.zeros_like(eye), np.zeros(0), np.zeros(0), X)
    assert not Y.any()
    # 'ones': rank one everywhere -> Y = 1 (1^T X)
    ones = np.ones(n * p)
    Y = oracle.hodlr_matvec(n, p, [1] * p, np.ones((1 << p) * b * b), ones, ones, X)
    assert relerr(Y, np.ones((n, 1)) * X.sum(axis=0)) < 1e-14


def test_identity_ones_hss():
    n, p = 256, 3
    b = n >> p
    nt, nb = (1 << p) - 2, (1 << p) - 1
    rng = np.random.default_rng(0)
    X = rng.standard_normal((n, 2))
    eye = np.tile(np.eye(b).ravel(), 1 << p)
    Y = oracle.hss_matvec(n, p, 0, eye, np.zeros(0), np.zeros(0), np.zeros(0), np.zeros(0), np.zeros(0), X)
    assert np.array_equal(Y, X)
    # ones: U = V = 1 (b x 1), R = W = [1; 1], B = [1], D = ones
    Y = oracle.hss_matvec(n, p, 1, np.ones((1 << p) * b * b), np.ones(n), np.ones(n), np.ones(2 * nt),
                          np.ones(2 * nt), np.ones(2 * nb), X)
    assert relerr(Y, np.ones((n, 1)) * X.sum(axis=0)) < 1e-14


# --------------------------------------------------------------- invariants --

def test_linearity_and_column_independence():
    rng = np.random.default_rng(5)
    n, p, ranks = 512, 3, [4, 4, 4]
    h = hm_inputs.hodlr_random(n, p, ranks, cid=9)
    s = hm_inputs.hss_random(n, p, 4, cid=9)
    X1, X2 = rng.standard_normal((n, 3)), rng.standard_normal((n, 3))
    al, be = 0.75, -1.5
    for f in (lambda X: oracle.hodlr_matvec(n, p, ranks, h.D, h.U, h.V, X),
              lambda X: oracle.hss_matvec(n, p, 4, s.D, s.U, s.V, s.R, s.W, s.B, X)):
        lhs = f(al * X1 + be * X2)
        rhs_ = al * f(X1) + be * f(X2)
        assert relerr(lhs, rhs_) < 1e-14
        full = f(X1)
        for j in range(3):  # every column is the nrhs = 1 run on that column, bit for bit
            assert np.array_equal(full[:, j], f(X1[:, j:j + 1])[:, 0])


def test_symmetry_inner_products():
    """Symmetric generators (U = V, W = R, B21 = B12^T, D_i symmetric) give A = A^T."""
    rng = np.random.default_rng(8)
    n, p, k = 256, 3, 3
    c = np.arange(1, 9) * 32
    D, U, V, R, W, B = random_hss_general(c, p, k, rng)
    D = D.reshape(-1, 32, 32); D = (D + D.transpose(0, 2, 1)).ravel()
    B = B.reshape(-1, 2, k, k); B[:, 1] = B[:, 0].transpose(0, 2, 1); B = B.ravel()
    x, y = rng.standard_normal((n, 1)), rng.standard_normal((n, 1))
    f = lambda X: oracle.hss_matvec(n, p, k, D, U, U, R, R, B, X)
    assert abs((x.T @ f(y)).item() - (y.T @ f(x)).item()) < 1e-12 * np.linalg.norm(f(x)) * np.linalg.norm(y)
    ranks = [k] * p
    Dh, Uh, _ = random_hodlr_general(c, p, ranks, rng)
    Dh = Dh.reshape(-1, 32, 32); Dh = (Dh + Dh.transpose(0, 2, 1)).ravel()
    # V_l = U_l: A(I_b,I_a) = U_l(I_b) U_l(I_a)^T = A(I_a,I_b)^T
    g = lambda X: oracle.hodlr_matvec(n, p, ranks, Dh, Uh, Uh, X)
    assert abs((x.T @ g(y)).item() - (y.T @ g(x)).item()) < 1e-12 * np.linalg.norm(g(x)) * np.linalg.norm(y)


def test_leaves_variants_equal_full_rows():
    n, p = 1024, 4
    b = n >> p
    ranks = [3, 2, 4, 1]
    h = hm_inputs.hodlr_random(n, p, ranks, cid=7)
    s = hm_inputs.hss_random(n, p, 5, cid=7)
    X = hm_inputs.rhs(n, 3, cid=7)
    leaves = [0, 5, 15, 5]
    Yf = oracle.hodlr_matvec(n, p, ranks, h.D, h.U, h.V, X)
    Dsel = np.concatenate([h.D[L * b * b:(L + 1) * b * b] for L in leaves])
    Yl = oracle.hodlr_matvec_leaves(n, p, ranks, Dsel, h.U, h.V, X, leaves)
    assert np.array_equal(Yl, np.concatenate([Yf[L * b:(L + 1) * b] for L in leaves]))
    Yf = oracle.hss_matvec(n, p, 5, s.D, s.U, s.V, s.R, s.W, s.B, X)
    Dsel = np.concatenate([s.D[L * b * b:(L + 1) * b * b] for L in leaves])
    Yl = oracle.hss_matvec_leaves(n, p, 5, Dsel, s.U, s.V, s.R, s.W, s.B, X, leaves)
    assert np.array_equal(Yl, np.concatenate([Yf[L * b:(L + 1) * b] for L in leaves]))


def test_thread_count_independence():
    """results bitwise independent of scheduling (1 thread vs all)."""
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r); import oracle, hm_inputs;"
        "h = hm_inputs.hodlr_random(1<<14, 5, [8]*5, cid=3); X = hm_inputs.rhs(1<<14, 2, cid=3);"
        "s = hm_inputs.hss_random(1<<13, 5, 8, cid=3); X2 = hm_inputs.rhs(1<<13, 2, cid=3);"
        "y = oracle.hodlr_matvec(1<<14, 5, h.ranks, h.D, h.U, h.V, X);"
        "z = oracle.hss_matvec(1<<13, 5, 8, s.D, s.U, s.V, s.R, s.W, s.B, X2);"
        "sys.stdout.buffer.write(y.tobytes() + z.tobytes())"
    ) % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for t in ("1", "4"):
        env = dict(os.environ, OMP_NUM_THREADS=t)
        outs.append(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, check=True).stdout)
    assert outs[0] == outs[1] and len(outs[0]) > 0


def test_invalid_arguments_rejected():
    with pytest.raises(ValueError):
        oracle.hodlr_matvec(8, 1, [1], np.zeros(32), np.zeros(8), np.zeros(8), np.zeros(8), c=[4, 3])
    with pytest.raises(ValueError):
        oracle.hss_matvec(8, 1, -1, np.zeros(32), np.zeros(0), np.zeros(0), np.zeros(0), np.zeros(0),
                          np.zeros(0), np.zeros(8))
