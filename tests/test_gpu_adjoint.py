"""GPU parity of the adjoint product Y = A^T X against the oracle.

Same bar as the forward product (BASELINE.json north_star): ||Y_gpu - Y_ref||_F /
||Y_ref||_F <= 1e-12 in fp64, on the same seeded inputs; small cases through the
full oracle (every shape family of test_gpu_parity: GEMV, DMMA and generic
paths, ragged column chunks, k = 0, p = 0), config 5 at full size against the
closed form (configs 3 and 4 in full: test_gpu_fullsize.py).
"""
import numpy as np
import pytest

import hm_inputs
import oracle
from test_gpu_parity import HODLR_CASES, HSS_CASES, TOL, dev, relerr, tridiag_residual

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hm():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1909_07909_b200 as hm_
    from paper_1909_07909_b200 import build
    build.build()
    hm_.load()
    return hm_


def gpu_hodlr_t(hm, h, X):
    Y = hm.hodlr_matvec_t(h.n, h.levels, h.leaf, h.ranks, dev(h.D), dev(h.U), dev(h.V), dev(X))
    torch.cuda.synchronize()
    return Y.cpu().numpy()


def gpu_hss_t(hm, s, X):
    Y = hm.hss_matvec_t(s.n, s.levels, s.leaf, s.k, dev(s.D), dev(s.U), dev(s.V), dev(s.R), dev(s.W), dev(s.B),
                        dev(X))
    torch.cuda.synchronize()
    return Y.cpu().numpy()


@pytest.mark.parametrize("n,leaf,levels,k,m", HODLR_CASES)
def test_hodlr_adjoint_vs_oracle(hm, n, leaf, levels, k, m):
    h = hm_inputs.hodlr_random(n, levels, [k] * levels, cid=31)
    X = hm_inputs.rhs(n, m, cid=31)
    Yr = oracle.hodlr_matvec_t(n, levels, h.ranks, h.D, h.U, h.V, X)
    assert relerr(gpu_hodlr_t(hm, h, X), Yr) <= TOL


@pytest.mark.parametrize("n,leaf,levels,k,m", HSS_CASES)
def test_hss_adjoint_vs_oracle(hm, n, leaf, levels, k, m):
    s = hm_inputs.hss_random(n, levels, k, cid=32)
    X = hm_inputs.rhs(n, m, cid=32)
    Yr = oracle.hss_matvec_t(n, levels, k, s.D, s.U, s.V, s.R, s.W, s.B, X)
    assert relerr(gpu_hss_t(hm, s, X), Yr) <= TOL


@pytest.mark.parametrize("level", [1, 4, 8])
def test_hodlr_adjoint_level_isolation(hm, level):
    """D = 0 and one level non-zero (G14), adjoint: only U_l^T X and V_l rows act."""
    n, p, k, m = 1 << 16, 8, 16, 8
    h = hm_inputs.hodlr_random(n, p, [k] * p, cid=33)
    h.D[:] = 0
    for l in range(1, p + 1):
        if l != level:
            h.V[h.level_slice(l)] = 0
    X = hm_inputs.rhs(n, m, cid=33)
    Yr = oracle.hodlr_matvec_t(n, p, h.ranks, h.D, h.U, h.V, X)
    assert np.linalg.norm(Yr) > 0
    assert relerr(gpu_hodlr_t(hm, h, X), Yr) <= TOL


@pytest.mark.parametrize("level", [1, 3, 6])
def test_hss_adjoint_level_isolation(hm, level):
    """D = 0, cores zero except one level (pins the transposed, swapped cores)."""
    n, p, k, m = 8192, 7, 16, 4
    s = hm_inputs.hss_random(n, p, k, cid=34)
    s.D[:] = 0
    B = s.B.reshape(-1, 2, k, k)
    B[:(1 << (level - 1)) - 1] = 0
    B[(1 << level) - 1:] = 0
    X = hm_inputs.rhs(n, m, cid=34)
    Yr = oracle.hss_matvec_t(n, p, k, s.D, s.U, s.V, s.R, s.W, s.B, X)
    assert np.linalg.norm(Yr) > 0
    assert relerr(gpu_hss_t(hm, s, X), Yr) <= TOL


def test_adjoint_inner_product_and_determinism(hm):
    """<Y, A X> = <A^T Y, X> with both products on the GPU; repeated calls bitwise equal."""
    n, p, k, m = 1 << 15, 7, 32, 8
    s = hm_inputs.hss_random(n, p, k, cid=35)
    g = [dev(a) for a in (s.D, s.U, s.V, s.R, s.W, s.B)]
    X, Z = dev(hm_inputs.rhs(n, m, cid=35)), dev(hm_inputs.rhs(n, m, cid=36))
    AX = hm.hss_matvec(n, p, s.leaf, k, *g, X)
    AtZ = hm.hss_matvec_t(n, p, s.leaf, k, *g, Z)
    AtZ2 = hm.hss_matvec_t(n, p, s.leaf, k, *g, Z)
    lhs, rhs = float((Z * AX).sum()), float((AtZ * X).sum())
    assert abs(lhs - rhs) <= 1e-12 * float(torch.linalg.norm(AX) * torch.linalg.norm(Z))
    assert torch.equal(AtZ, AtZ2)


# ------------------------------------------------- full-size configs --

def test_config5_adjoint_closed_form(hm):
    """The inverse Laplacian is symmetric: A^T X is the closed form, at n = 2^24."""
    cfg = hm_inputs.CONFIGS[5]
    hd = hm_inputs.hodlr_inverse_laplacian(cfg.n, cfg.levels, xp=torch, device="cuda:0")
    X = hm_inputs.rhs(cfg.n, 1, cid=5)
    Y = hm.hodlr_matvec_t(cfg.n, cfg.levels, cfg.leaf, hd.ranks, hd.D, hd.U, hd.V, dev(X))
    torch.cuda.synchronize()
    Y = Y.cpu().numpy()
    assert relerr(Y, oracle.laplacian_inverse_apply(X)) <= TOL
    assert tridiag_residual(Y, X) <= 1e-14
