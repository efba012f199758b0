"""Randomised GPU parity sweep: seeded random shapes (leaf size, depth, ranks, nrhs,
forward / adjoint, uniform / general trees) against the oracle, so that every
dispatch branch of the C-ABI (GEMV, DMMA, TMA, generic, small-tree, general-tree
kernels) meets shapes nobody picked by hand. Tolerance 1e-12 (BASELINE.json).
"""
import numpy as np
import pytest

import hm_inputs
import oracle
from test_gpu_parity import TOL, dev, relerr
from test_gpu_general import ragged_tree
from test_oracle import random_hodlr_general, random_hss_general

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

LEAVES = [1, 7, 16, 32, 48, 64, 100, 128, 192, 256]
RANKS = [0, 1, 2, 3, 5, 8, 16, 24, 32, 64]
NRHS = [1, 2, 3, 7, 8, 16, 17, 32, 33]


@pytest.fixture(scope="module")
def hm():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1909_07909_b200 as hm_
    from paper_1909_07909_b200 import build
    build.build()
    hm_.load()
    return hm_


def cases(seed, count):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        b = int(rng.choice(LEAVES))
        p = int(rng.integers(0, 9))
        if b << p > 40000:
            continue
        k = int(rng.choice(RANKS))
        m = int(rng.choice(NRHS))
        op = int(rng.integers(0, 2))
        out.append((b, p, k, m, op))
    return out


@pytest.mark.parametrize("b,p,k,m,op", cases(2026, 64))
def test_random_hodlr(hm, b, p, k, m, op):
    n = b << p
    h = hm_inputs.hodlr_random(n, p, [k] * p, cid=81)
    X = hm_inputs.rhs(n, m, cid=81)
    f = hm.hodlr_matvec_t if op else hm.hodlr_matvec
    Y = f(n, p, b, h.ranks, dev(h.D), dev(h.U), dev(h.V), dev(X))
    torch.cuda.synchronize()
    ref = (oracle.hodlr_matvec_t if op else oracle.hodlr_matvec)(n, p, h.ranks, h.D, h.U, h.V, X)
    assert relerr(Y.cpu().numpy(), ref) <= TOL


@pytest.mark.parametrize("b,p,k,m,op", cases(1909, 64))
def test_random_hss(hm, b, p, k, m, op):
    n = b << p
    s = hm_inputs.hss_random(n, p, k, cid=82)
    X = hm_inputs.rhs(n, m, cid=82)
    f = hm.hss_matvec_t if op else hm.hss_matvec
    g = [dev(a) for a in (s.D, s.U, s.V, s.R, s.W, s.B)]
    Y = f(n, p, b, k, *g, dev(X))
    torch.cuda.synchronize()
    ref = (oracle.hss_matvec_t if op else oracle.hss_matvec)(n, p, k, s.D, s.U, s.V, s.R, s.W, s.B, X)
    assert relerr(Y.cpu().numpy(), ref) <= TOL


@pytest.mark.parametrize("seed", range(16))
def test_random_general_trees(hm, seed):
    rng = np.random.default_rng(900 + seed)
    p = int(rng.integers(1, 8))
    n = int(rng.integers(1 << p, 6000))
    c = ragged_tree(n, p, seed, empty=float(rng.uniform(0, 0.3)))
    ranks = [int(v) for v in rng.integers(0, 12, size=p)]
    m = int(rng.choice([1, 3, 9]))
    D, U, V = random_hodlr_general(c, p, ranks, rng)
    X = rng.standard_normal((n, m))
    for op in (0, 1):
        Y = hm.hodlr_matvec_general(n, p, c, ranks, dev(D), dev(U), dev(V), dev(X), op=op)
        torch.cuda.synchronize()
        ref = (oracle.hodlr_matvec_t if op else oracle.hodlr_matvec)(n, p, ranks, D, U, V, X, c=c)
        assert relerr(Y.cpu().numpy(), ref) <= TOL
    k = int(rng.choice([0, 2, 16, 32]))
    D, U, V, R, W, B = random_hss_general(c, p, k, rng)
    for op in (0, 1):
        Y = hm.hss_matvec_general(n, p, c, k, *[dev(a) for a in (D, U, V, R, W, B)], dev(X), op=op)
        torch.cuda.synchronize()
        ref = (oracle.hss_matvec_t if op else oracle.hss_matvec)(n, p, k, D, U, V, R, W, B, X, c=c)
        assert relerr(Y.cpu().numpy(), ref) <= TOL


@pytest.mark.parametrize("seed", range(12))
def test_random_ragged_wide(hm, seed):
    """Random ragged trees with ranks that are multiples of 8 on most levels and nrhs
    2..40: the 128-bit-fragment DMMA leaf pass (gen_leaf_mma_al) and the one-tile
    V^T X meet random leaf sizes, alignments and column chunks."""
    rng = np.random.default_rng(1300 + seed)
    p = int(rng.integers(3, 8))
    n = int(rng.integers(8 << p, 12000))
    c = ragged_tree(n, p, 50 + seed, empty=float(rng.uniform(0, 0.2)))
    ranks = [int(rng.choice([8, 16, 16, 32, 3, 0])) for _ in range(p)]
    m = int(rng.integers(2, 41))
    D, U, V = random_hodlr_general(c, p, ranks, rng)
    X = rng.standard_normal((n, m))
    Y = hm.hodlr_matvec_general(n, p, c, ranks, dev(D), dev(U), dev(V), dev(X), op=0)
    torch.cuda.synchronize()
    assert relerr(Y.cpu().numpy(), oracle.hodlr_matvec(n, p, ranks, D, U, V, X, c=c)) <= TOL


@pytest.mark.parametrize("seed", range(12))
def test_random_hss_per_level_ranks(hm, seed):
    """Random per-level HSS ranks (multiples of 8 take the DMMA level kernels and the
    cooperative small-level sweep, others the CUDA-core kernels), random nrhs and
    operator, every row against the oracle."""
    rng = np.random.default_rng(1400 + seed)
    p = int(rng.integers(2, 10))
    b = int(rng.choice([32, 64, 128]))
    n = b << p
    ranks = [int(rng.choice([8, 16, 24, 32, 5, 12])) for _ in range(p)]
    m = int(rng.integers(2, 35))
    op = int(rng.integers(0, 2))
    s = hm_inputs.hss_random_ranked(n, p, ranks, cid=1400 + seed)
    X = hm_inputs.rhs(n, m, cid=1400 + seed)
    g = [dev(a) for a in (s.D, s.U, s.V, s.R, s.W, s.B)]
    Y = hm.hss_matvec_ranked(n, p, b, ranks, *g, dev(X), op=op)
    torch.cuda.synchronize()
    ref = oracle.hss_matvec_ranked(n, p, ranks, s.D, s.U, s.V, s.R, s.W, s.B, X, trans=bool(op))
    assert relerr(Y.cpu().numpy(), ref) <= TOL
