"""Pins for the oracle's SURVEY §8(f) routines (adjoint, norm estimate, hss2hodlr).

Each check compares the oracle with something fixed independently of it:
dense brute force built in numpy from the definitions (Def. 2.2 P:213-222,
eq. (3)) and transposed with numpy, the inner-product identity
<y, A x> = <A^T y, x>, symmetric generators (A^T = A exactly), the closed-form
spectral norm of the inverse 1D Laplacian, dense SVD, and the monotonicity of
the power method on A A^* (P:1146).
"""
import numpy as np
import pytest

import hm_inputs
import oracle
from test_oracle import dense_hodlr_np, dense_hss_np, random_hodlr_general, random_hss_general, relerr, tree_sets

GENERAL_TREES = [
    # c (leaf endpoints), p, hodlr ranks, hss rank
    (np.arange(1, 17) * 32, 4, [4, 3, 2, 5], 4),          # uniform
    (np.array([3, 7, 7, 20, 26, 26, 31, 40]), 3, [2, 1, 3], 2),  # ragged, empty leaves (Fig. 4 style)
    (np.array([5, 9]), 1, [0], 3),                         # p = 1, rank-0 level
    (np.array([17]), 0, [], 2),                            # p = 0: A = D
]


@pytest.mark.parametrize("c,p,ranks,k", GENERAL_TREES)
def test_hodlr_adjoint_vs_dense_transpose(c, p, ranks, k):
    rng = np.random.default_rng(21)
    n = int(c[-1])
    D, U, V = random_hodlr_general(c, p, ranks, rng)
    X = rng.standard_normal((n, 3))
    A = dense_hodlr_np(n, p, ranks, D, U, V, c)
    Y = oracle.hodlr_matvec_t(n, p, ranks, D, U, V, X, c=c)
    assert relerr(Y, A.T @ X) < 1e-14


@pytest.mark.parametrize("c,p,ranks,k", GENERAL_TREES)
def test_hss_adjoint_vs_dense_transpose(c, p, ranks, k):
    rng = np.random.default_rng(22)
    n = int(c[-1])
    D, U, V, R, W, B = random_hss_general(c, p, k, rng)
    X = rng.standard_normal((n, 2))
    A = dense_hss_np(n, p, k, D, U, V, R, W, B, c)
    Y = oracle.hss_matvec_t(n, p, k, D, U, V, R, W, B, X, c=c)
    assert relerr(Y, A.T @ X) < 1e-14


def test_adjoint_config_shapes_inner_product():
    """<Y, A X> = <A^T Y, X> on BASELINE config-1 / config-2 generators."""
    c1, c2 = hm_inputs.CONFIGS[1], hm_inputs.CONFIGS[2]
    h = hm_inputs.hodlr_random(c1.n, c1.levels, [c1.k] * c1.levels, cid=1)
    s = hm_inputs.hss_random(c2.n, c2.levels, c2.k, cid=2)
    rng = np.random.default_rng(23)
    for n, f, ft in (
        (c1.n, lambda X: oracle.hodlr_matvec(c1.n, c1.levels, h.ranks, h.D, h.U, h.V, X),
         lambda X: oracle.hodlr_matvec_t(c1.n, c1.levels, h.ranks, h.D, h.U, h.V, X)),
        (c2.n, lambda X: oracle.hss_matvec(c2.n, c2.levels, c2.k, s.D, s.U, s.V, s.R, s.W, s.B, X),
         lambda X: oracle.hss_matvec_t(c2.n, c2.levels, c2.k, s.D, s.U, s.V, s.R, s.W, s.B, X)),
    ):
        X, Yv = rng.standard_normal((n, 4)), rng.standard_normal((n, 4))
        lhs = np.sum(Yv * f(X))
        rhs = np.sum(ft(Yv) * X)
        assert abs(lhs - rhs) <= 1e-13 * np.linalg.norm(f(X)) * np.linalg.norm(Yv)


def test_adjoint_of_symmetric_is_forward_bitwise():
    """U = V (W = R, B21 = B12^T), D_i symmetric: A^T = A, and the adjoint runs the
    same products on equal values in the same order, so the results are identical."""
    rng = np.random.default_rng(24)
    n, p, k = 256, 3, 3
    c = np.arange(1, 9) * 32
    D, U, V, R, W, B = random_hss_general(c, p, k, rng)
    D = D.reshape(-1, 32, 32); D = (D + D.transpose(0, 2, 1)).ravel()
    B = B.reshape(-1, 2, k, k); B[:, 1] = B[:, 0].transpose(0, 2, 1); B = B.ravel()
    X = rng.standard_normal((n, 2))
    assert np.array_equal(oracle.hss_matvec_t(n, p, k, D, U, U, R, R, B, X),
                          oracle.hss_matvec(n, p, k, D, U, U, R, R, B, X))
    ranks = [k] * p
    Dh, Uh, _ = random_hodlr_general(c, p, ranks, rng)
    Dh = Dh.reshape(-1, 32, 32); Dh = (Dh + Dh.transpose(0, 2, 1)).ravel()
    assert np.array_equal(oracle.hodlr_matvec_t(n, p, ranks, Dh, Uh, Uh, X),
                          oracle.hodlr_matvec(n, p, ranks, Dh, Uh, Uh, X))


def test_adjoint_inverse_laplacian_closed_form():
    """The inverse Laplacian is symmetric: A^T X = A X = the O(n) closed form."""
    n, p = 4096, 4
    h = hm_inputs.hodlr_inverse_laplacian(n, p)
    X = hm_inputs.rhs(n, 2, cid=5)
    assert relerr(oracle.hodlr_matvec_t(n, p, h.ranks, h.D, h.U, h.V, X), oracle.laplacian_inverse_apply(X)) < 1e-14
    s = hm_inputs.hss_inverse_laplacian(n, p)
    assert relerr(oracle.hss_matvec_t(n, p, s.k, s.D, s.U, s.V, s.R, s.W, s.B, X),
                  oracle.laplacian_inverse_apply(X)) < 1e-14


def test_adjoint_leaves_variants_equal_full_rows():
    n, p = 1024, 4
    b = n >> p
    h = hm_inputs.hodlr_random(n, p, [3, 2, 4, 1], cid=7)
    s = hm_inputs.hss_random(n, p, 5, cid=7)
    X = hm_inputs.rhs(n, 3, cid=7)
    leaves = [0, 6, 15]
    Yf = oracle.hodlr_matvec_t(n, p, h.ranks, h.D, h.U, h.V, X)
    Dsel = np.concatenate([h.D[L * b * b:(L + 1) * b * b] for L in leaves])
    Yl = oracle.hodlr_matvec_t_leaves(n, p, h.ranks, Dsel, h.U, h.V, X, leaves)
    assert np.array_equal(Yl, np.concatenate([Yf[L * b:(L + 1) * b] for L in leaves]))
    Yf = oracle.hss_matvec_t(n, p, 5, s.D, s.U, s.V, s.R, s.W, s.B, X)
    Dsel = np.concatenate([s.D[L * b * b:(L + 1) * b * b] for L in leaves])
    Yl = oracle.hss_matvec_t_leaves(n, p, 5, Dsel, s.U, s.V, s.R, s.W, s.B, X, leaves)
    assert np.array_equal(Yl, np.concatenate([Yf[L * b:(L + 1) * b] for L in leaves]))


# ---------------------------------------------------------- norm estimate --

def test_norm2_est_diagonal_and_zero():
    """S:165-173 examples: diag(1,2,3) -> ~3 within 1%; the zero operator -> 0."""
    D = np.diag([1.0, 2.0, 3.0]).ravel()
    x0 = np.array([1.0, 1.0, 1.0])
    est = oracle.hodlr_norm2_est(3, 0, [], D, np.zeros(0), np.zeros(0), x0, 20)
    assert abs(est - 3.0) <= 0.01 * 3.0 and est <= 3.0
    z = oracle.hodlr_norm2_est(64, 2, [2, 2], np.zeros(4 * 16 * 16), np.zeros(64 * 4), np.zeros(64 * 4),
                               np.ones(64), 5)
    assert z == 0.0


@pytest.mark.parametrize("fmt", ["hodlr", "hss"])
def test_norm2_est_inverse_laplacian_closed_form(fmt):
    """||T^{-1}||_2 = 1 / (2 - 2 cos(pi/(n+1))) (smallest eigenvalue of tridiag(-1,2,-1));
    the top eigenvalue is separated (ratio 1/4), so 40 steps reach rounding level.
    2 - 2cos(x) = 4 sin^2(x/2), written without the cancellation."""
    n, p = 2048, 4
    exact = 1.0 / (4.0 * np.sin(np.pi / (2 * (n + 1))) ** 2)
    x0 = hm_inputs.rhs(n, 1, cid=5).ravel()
    if fmt == "hodlr":
        h = hm_inputs.hodlr_inverse_laplacian(n, p)
        est = oracle.hodlr_norm2_est(n, p, h.ranks, h.D, h.U, h.V, x0, 40)
    else:
        s = hm_inputs.hss_inverse_laplacian(n, p)
        est = oracle.hss_norm2_est(n, p, s.k, s.D, s.U, s.V, s.R, s.W, s.B, x0, 40)
    assert abs(est - exact) <= 1e-12 * exact


def test_norm2_est_random_vs_svd_and_monotone():
    """Random operators: eta <= sigma_1 always (||A^* v|| for unit v), within 5% of the
    dense-SVD sigma_1 after the budget, and nondecreasing in the iteration count."""
    rng = np.random.default_rng(25)
    n, p, k = 256, 3, 4
    c = np.arange(1, 9) * 32
    ranks = [k] * p
    for trial in range(5):
        D, U, V = random_hodlr_general(c, p, ranks, rng)
        A = dense_hodlr_np(n, p, ranks, D, U, V, c)
        s1 = np.linalg.svd(A, compute_uv=False)[0]
        x0 = rng.standard_normal(n)
        ests = [oracle.hodlr_norm2_est(n, p, ranks, D, U, V, x0, it) for it in (1, 2, 5, 20, 200)]
        assert all(e <= s1 * (1 + 1e-13) for e in ests)
        assert all(b >= a * (1 - 1e-14) for a, b in zip(ests, ests[1:]))
        assert ests[-1] >= 0.95 * s1
        Dh, Uh, Vh, Rh, Wh, Bh = random_hss_general(c, p, k, rng)
        Ah = dense_hss_np(n, p, k, Dh, Uh, Vh, Rh, Wh, Bh, c)
        s1h = np.linalg.svd(Ah, compute_uv=False)[0]
        e = oracle.hss_norm2_est(n, p, k, Dh, Uh, Vh, Rh, Wh, Bh, x0, 200)
        assert e <= s1h * (1 + 1e-13) and e >= 0.95 * s1h


# -------------------------------------------------------------- hss2hodlr --

@pytest.mark.parametrize("c,p,k", [(np.arange(1, 17) * 32, 4, 4), (np.array([3, 7, 7, 20, 26, 26, 31, 40]), 3, 2),
                                   (np.array([6, 11]), 1, 3)])
def test_hss_to_hodlr_vs_dense(c, p, k):
    """hss2hodlr is exact: the HODLR matrix built from the converted factors
    (numpy, Def. 2.2) equals the HSS matrix built from eq. (3) (numpy)."""
    rng = np.random.default_rng(26)
    n = int(c[-1])
    D, U, V, R, W, B = random_hss_general(c, p, k, rng)
    Uh, Vh = oracle.hss_to_hodlr(n, p, k, U, V, R, W, B, c=c)
    Ah = dense_hodlr_np(n, p, [k] * p, D, Uh, Vh, c)
    As = dense_hss_np(n, p, k, D, U, V, R, W, B, c)
    assert relerr(Ah, As) < 1e-14


def test_hss_to_hodlr_factors_match_nested_bases():
    """V_l = V^(l) (eq. (3) bases, built in numpy here) and U_l(I_a) = U^(l)_a S_{a,sib a}."""
    rng = np.random.default_rng(27)
    n, p, k = 256, 3, 3
    c = np.arange(1, 9) * 32
    D, U, V, R, W, B = random_hss_general(c, p, k, rng)
    Uh, Vh = oracle.hss_to_hodlr(n, p, k, U, V, R, W, B)
    Rr, Wr, Br = R.reshape(-1, 2 * k, k), W.reshape(-1, 2 * k, k), B.reshape(-1, 2, k, k)
    Ub, Vb = U.reshape(n, k).copy(), V.reshape(n, k).copy()
    for l in range(p, 0, -1):
        sets = tree_sets(c, p, l)
        Ul = np.empty((n, k))
        for a in range(1 << l):
            lo, hi = sets[a]
            Ul[lo:hi] = Ub[lo:hi] @ Br[(1 << (l - 1)) - 1 + (a >> 1), a & 1]
        assert relerr(Uh[(l - 1) * n * k:l * n * k].reshape(n, k), Ul) < 1e-14
        assert relerr(Vh[(l - 1) * n * k:l * n * k].reshape(n, k), Vb) < 1e-14
        if l > 1:
            Un, Vn = np.empty((n, k)), np.empty((n, k))
            for i in range(1 << (l - 1)):
                node = (1 << (l - 1)) - 2 + i
                for ch in range(2):
                    lo, hi = sets[2 * i + ch]
                    Un[lo:hi] = Ub[lo:hi] @ Rr[node, ch * k:(ch + 1) * k]
                    Vn[lo:hi] = Vb[lo:hi] @ Wr[node, ch * k:(ch + 1) * k]
            Ub, Vb = Un, Vn
