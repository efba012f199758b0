"""GPU parity on general cluster trees and per-level HODLR ranks.

Trees given by leaf endpoint vectors: ragged leaves, empty leaves
(Fig. 4), the default ceil split of P:378-379 for n not a multiple
of 2^p, and nodes big enough to be split over several V^T X chunks. Forward
and adjoint products against the oracle at 1e-12 (BASELINE.json north_star).
"""
import numpy as np
import pytest

import oracle
from test_gpu_parity import TOL, dev, relerr
from test_oracle import random_hodlr_general, random_hss_general

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


def ragged_tree(n, p, seed, empty=0.15):
    """Random nondecreasing endpoints with about `empty` of the leaves empty."""
    rng = np.random.default_rng(seed)
    w = rng.uniform(0.2, 1.8, size=1 << p)
    w[rng.uniform(size=1 << p) < empty] = 0.0
    c = np.floor(np.cumsum(w) / w.sum() * n).astype(np.int64)
    c[-1] = n
    return c


TREES = [
    ("fig4", np.array([3, 7, 7, 20, 26, 26, 31, 40]), 3),
    ("ceil_split_1000", None, None),            # default cluster n = 1000, nmin = 64
    ("ragged_p6", ragged_tree(6000, 6, 1), 6),
    ("ragged_p9", ragged_tree(40000, 9, 2), 9),
    ("big_nodes", np.array([9000, 20000, 20000, 31000]), 2),   # nodes > one 4096-row chunk
    ("p0", np.array([77]), 0),
]


def tree(name, c, p):
    if c is None:
        p, c = oracle.default_cluster(1000, 64)
    return int(c[-1]), p, np.asarray(c, dtype=np.int64)


@pytest.mark.parametrize("name,c,p", TREES)
@pytest.mark.parametrize("m", [1, 5, 16])
def test_hodlr_general_vs_oracle(hm, name, c, p, m):
    n, p, c = tree(name, c, p)
    rng = np.random.default_rng(51 + m)
    ranks = [int(v) for v in rng.integers(0, 17, size=p)]  # per-level ranks incl. 0
    D, U, V = random_hodlr_general(c, p, ranks, rng)
    X = rng.standard_normal((n, m))
    for op in (0, 1):
        Y = hm.hodlr_matvec_general(n, p, c, ranks, dev(D), dev(U), dev(V), dev(X), op=op)
        torch.cuda.synchronize()
        f = oracle.hodlr_matvec_t if op else oracle.hodlr_matvec
        assert relerr(Y.cpu().numpy(), f(n, p, ranks, D, U, V, X, c=c)) <= TOL, op


@pytest.mark.parametrize("name,c,p", TREES)
@pytest.mark.parametrize("k,m,kernel", [(16, 1, "gen_vt_gemv"), (2, 1, "gen_vt_gemv"), (64, 1, "gen_vt_gemv"),
                                        (16, 2, "gen_vt_mma"), (32, 9, "gen_vt_mma"), (64, 33, "gen_vt_mma"),
                                        (16, 40, "gen_vt_mma")])
def test_hodlr_general_one_rank_tuned_vt(hm, name, c, p, k, m, kernel):
    """One rank on every level of a general tree: V^T X per chunk runs the
    streaming GEMV (m = 1) or DMMA (k in 16/32/64) chunk kernel; ragged chunk
    ends read as zero."""
    n, p, c = tree(name, c, p)
    if p == 0:
        pytest.skip("no off-diagonal levels")
    rng = np.random.default_rng(81 + k + m)
    ranks = [k] * p
    D, U, V = random_hodlr_general(c, p, ranks, rng)
    X = rng.standard_normal((n, m))
    hm.hm_profile_collect()
    hm.hm_profile_enable(True)
    for op in (0, 1):
        Y = hm.hodlr_matvec_general(n, p, c, ranks, dev(D), dev(U), dev(V), dev(X), op=op)
        torch.cuda.synchronize()
        f = oracle.hodlr_matvec_t if op else oracle.hodlr_matvec
        assert relerr(Y.cpu().numpy(), f(n, p, ranks, D, U, V, X, c=c)) <= TOL, op
    hm.hm_profile_enable(False)
    names = {t[0] for t in hm.hm_profile_collect()}
    assert kernel in names, names


@pytest.mark.parametrize("name,c,p", TREES)
@pytest.mark.parametrize("k,m", [(4, 1), (16, 16), (32, 3), (0, 2)])
def test_hss_general_vs_oracle(hm, name, c, p, k, m):
    n, p, c = tree(name, c, p)
    rng = np.random.default_rng(61 + k + m)
    D, U, V, R, W, B = random_hss_general(c, p, k, rng)
    X = rng.standard_normal((n, m))
    g = [dev(a) for a in (D, U, V, R, W, B)]
    for op in (0, 1):
        Y = hm.hss_matvec_general(n, p, c, k, *g, dev(X), op=op)
        torch.cuda.synchronize()
        f = oracle.hss_matvec_t if op else oracle.hss_matvec
        assert relerr(Y.cpu().numpy(), f(n, p, k, D, U, V, R, W, B, X, c=c)) <= TOL, op


@pytest.mark.parametrize("n,leaf,p,ranks,m,route", [
    (65536, 256, 8, [64, 32, 16, 8, 4, 2, 1, 0], 8, "uniform"),   # ranks < 8: generic leaf pass
    (16384, 64, 8, [1, 2, 3, 4, 5, 6, 7, 8], 3, "uniform"),       # odd ranks: vt_contract groups
    (12288, 96, 7, [8, 16, 4, 2, 16, 8, 1], 2, "general"),        # leaf not a multiple of 64
    (4096, 1024, 2, [16, 8], 5, "general"),                       # fewer than 8 leaves
])
def test_uniform_tree_per_level_ranks(hm, n, leaf, p, ranks, m, route):
    """hodlr_matvec / hodlr_matvec_t on per-level ranks outside the tuned
    kernels' shapes: mixed tuned / generic uniform-tree kernels, or the
    general-tree kernels when the tree has no 8-leaf tiles of 64-multiples."""
    rng = np.random.default_rng(71)
    c = np.arange(1, (1 << p) + 1, dtype=np.int64) * leaf
    D, U, V = random_hodlr_general(c, p, ranks, rng)
    X = rng.standard_normal((n, m))
    hm.hm_profile_collect()
    hm.hm_profile_enable(True)
    Y = hm.hodlr_matvec(n, p, leaf, ranks, dev(D), dev(U), dev(V), dev(X))
    Yt = hm.hodlr_matvec_t(n, p, leaf, ranks, dev(D), dev(U), dev(V), dev(X))
    torch.cuda.synchronize()
    hm.hm_profile_enable(False)
    names = {t[0] for t in hm.hm_profile_collect()}
    assert any(nm.startswith("gen_") for nm in names) == (route == "general"), names
    assert relerr(Y.cpu().numpy(), oracle.hodlr_matvec(n, p, ranks, D, U, V, X)) <= TOL
    assert relerr(Yt.cpu().numpy(), oracle.hodlr_matvec_t(n, p, ranks, D, U, V, X)) <= TOL


@pytest.mark.parametrize("n,leaf,p,ranks,m", [
    (65536, 256, 8, [16, 8, 16, 4, 2, 16, 32, 1], 1),
    (131072, 256, 9, [1, 2, 4, 8, 16, 32, 64, 1, 0], 1),
    (32768, 128, 8, [2, 1, 2, 1, 2, 1, 2, 1], 1),
    (65536, 128, 9, [32, 16, 0, 64, 16, 32, 16, 16, 32], 8),
    (32768, 64, 9, [16, 32, 16, 32, 16, 32, 16, 32, 64], 2),
    (65536, 256, 8, [16, 32, 16, 32, 16, 32, 0, 32], 64),
    (16384, 64, 8, [64, 16, 16, 16, 32, 16, 16, 16], 13),
    (65536, 256, 8, [16, 8, 16, 8, 16, 8, 16, 8], 8),   # bench sweep's 16/8 set, smaller depth
    (65536, 128, 9, [8, 4, 2, 1, 0, 1, 2, 4, 8], 3),    # small ranks: DMMA V^T X, generic leaf pass
])
def test_uniform_tree_per_level_ranks_tuned_kernels(hm, n, leaf, p, ranks, m):
    """Per-level ranks that fit the tuned kernels run on them (one V^T X pass
    per distinct rank, per-segment ranks in the leaf pass), not on the general ones."""
    rng = np.random.default_rng(73 + m)
    c = np.arange(1, (1 << p) + 1, dtype=np.int64) * leaf
    D, U, V = random_hodlr_general(c, p, ranks, rng)
    X = rng.standard_normal((n, m))
    g = [dev(a) for a in (D, U, V)]
    hm.hm_profile_collect()
    hm.hm_profile_enable(True)
    Y = hm.hodlr_matvec(n, p, leaf, ranks, *g, dev(X))
    Yt = hm.hodlr_matvec_t(n, p, leaf, ranks, *g, dev(X))
    torch.cuda.synchronize()
    hm.hm_profile_enable(False)
    names = {t[0] for t in hm.hm_profile_collect()}
    assert not any(nm.startswith("gen_") for nm in names), names
    assert names & {"vt_gemv", "vt_mma_levels", "vt_lv"}, names
    assert relerr(Y.cpu().numpy(), oracle.hodlr_matvec(n, p, ranks, D, U, V, X)) <= TOL
    assert relerr(Yt.cpu().numpy(), oracle.hodlr_matvec_t(n, p, ranks, D, U, V, X)) <= TOL
    # bitwise repeatable (fixed-order reductions)
    Y2 = hm.hodlr_matvec(n, p, leaf, ranks, *g, dev(X))
    assert torch.equal(Y, Y2)


def test_per_level_ranks_hostio_matches_device(hm):
    """Per-level ranks through the host-buffer entry point (hodlr_matvec_hostio, the
    bench's e2e path) give bitwise the device-buffer result."""
    n, p, b, m = 65536, 8, 256, 8
    ranks = [16, 8, 16, 32, 8, 16, 4, 16]
    rng = np.random.default_rng(74)
    c = np.arange(1, (1 << p) + 1, dtype=np.int64) * b
    D, U, V = random_hodlr_general(c, p, ranks, rng)
    X = rng.standard_normal((n, m))
    g = [dev(a) for a in (D, U, V)]
    Yd = hm.hodlr_matvec(n, p, b, ranks, *g, dev(X)).cpu()
    Xh = torch.from_numpy(X).pin_memory()
    Yh = torch.empty_like(Xh).pin_memory()
    hm.hodlr_matvec_hostio(n, p, b, ranks, *g, Xh, Yh)
    torch.cuda.synchronize()
    assert torch.equal(Yh, Yd)
    assert relerr(Yh.numpy(), oracle.hodlr_matvec(n, p, ranks, D, U, V, X)) <= TOL


def test_general_uniform_endpoints_match_uniform_path(hm):
    """The general kernels on uniform endpoints agree with the tuned uniform kernels."""
    n, p, b, k, m = 32768, 7, 256, 16, 8
    rng = np.random.default_rng(72)
    c = np.arange(1, (1 << p) + 1, dtype=np.int64) * b
    D, U, V = random_hodlr_general(c, p, [k] * p, rng)
    X = dev(rng.standard_normal((n, m)))
    Yg = hm.hodlr_matvec_general(n, p, c, [k] * p, dev(D), dev(U), dev(V), X)
    Yu = hm.hodlr_matvec(n, p, b, [k] * p, dev(D), dev(U), dev(V), X)
    assert float(torch.linalg.norm(Yg - Yu) / torch.linalg.norm(Yu)) <= TOL
    Yg2 = hm.hodlr_matvec_general(n, p, c, [k] * p, dev(D), dev(U), dev(V), X)
    assert torch.equal(Yg, Yg2)


@pytest.mark.parametrize("m", [2, 8, 16, 32])
@pytest.mark.parametrize("dshift", [0, 1])
def test_ragged_wide_fragments(hm, m, dshift):
    """The nrhs >= 2 ragged leaf pass loads D and U as 128-bit fragments where the
    row address allows it (gen_leaf_mma_al_kernel): odd and even leaf sizes (rows of
    alternating 16-byte alignment), D starting 8 bytes past a 16-byte boundary
    (dshift = 1), levels whose rank is a multiple of 8 (the 128-bit U groups) next to
    ranks that are not (the 64-bit fallback columns). Every row against the oracle."""
    rng = np.random.default_rng(300 + m + 7 * dshift)
    p = 7
    sizes = rng.integers(60, 140, size=1 << p)
    sizes[::5] = 1                      # one-row leaves
    sizes[3::11] = 0                    # empty leaves
    c = np.cumsum(sizes).astype(np.int64)
    n = int(c[-1])
    ranks = [8, 16, 5, 0, 24, 3, 16]
    D, U, V = random_hodlr_general(c, p, ranks, rng)
    X = rng.standard_normal((n, m))
    Dbuf = torch.zeros(D.size + 1, dtype=torch.float64, device="cuda:0")
    Dbuf[dshift:dshift + D.size] = dev(D.ravel())
    Dd = Dbuf[dshift:dshift + D.size]
    Y, names = None, set()
    hm.hm_profile_collect()
    hm.hm_profile_enable(True)
    try:
        Y = hm.hodlr_matvec_general(n, p, c, ranks, Dd, dev(U), dev(V), dev(X), op=0)
        torch.cuda.synchronize()
    finally:
        hm.hm_profile_enable(False)
    names = {t[0] for t in hm.hm_profile_collect()}
    assert "gen_leaf_mma" in names, names
    assert relerr(Y.cpu().numpy(), oracle.hodlr_matvec(n, p, ranks, D, U, V, X, c=c)) <= TOL
