"""GPU parity of the HSS product with per-level and per-node ranks (
P:264) through the C-ABI (hss_matvec_ranked, hss_matvec_noderanked), A and A^T, against
the oracle's products (pinned in test_oracle_ranked.py). Tolerance: north_star's 1e-12."""
import numpy as np
import pytest

import hm_inputs
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module")
def hm():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1909_07909_b200 as hm_
    from paper_1909_07909_b200 import build
    build.build()
    hm_.load()
    return hm_


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda:0")


def relerr(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


CASES = [
    # n, levels, ranks (level 1..p), nrhs
    (1024, 4, [3, 5, 7, 8], 1),
    (1024, 4, [8, 7, 5, 3], 3),
    (4096, 6, [16, 16, 8, 8, 4, 4], 16),
    (8192, 7, [32, 16, 16, 16, 16, 32, 32], 8),       # leaf level k = 32: tuned Step 1 / Step 4 (DMMA)
    (8192, 7, [4, 8, 0, 8, 16, 16, 16], 1),           # a rank-0 level; m = 1 GEMV leaf kernels
    (1 << 15, 8, [64, 48, 32, 32, 16, 16, 16, 16], 32),
    (4096, 6, [5, 5, 5, 5, 5, 5], 2),                 # equal ranks: the tuned uniform path
    (256, 1, [6], 4),                                 # p = 1
]


@pytest.mark.parametrize("op", [0, 1])
@pytest.mark.parametrize("n,p,ranks,m", CASES)
def test_hss_ranked_vs_oracle(hm, n, p, ranks, m, op):
    s = hm_inputs.hss_random_ranked(n, p, ranks, cid=50)
    X = hm_inputs.rhs(n, m, cid=50)
    g = [dev(a) for a in (s.D, s.U, s.V, s.R, s.W, s.B)]
    Y = hm.hss_matvec_ranked(n, p, n >> p, ranks, *g, dev(X), op=op)
    torch.cuda.synchronize()
    Yr = oracle.hss_matvec_ranked(n, p, ranks, s.D, s.U, s.V, s.R, s.W, s.B, X, trans=bool(op))
    assert relerr(Y.cpu().numpy(), Yr) <= TOL


def test_hss_ranked_config4_tree(hm):
    """The config-4 tree (n = 2^22, leaf 128, 15 levels) with ranks growing towards the
    root (16 at the leaves, 32 on the middle levels, 48 on the top ones), nrhs 32: every row."""
    cfg = hm_inputs.CONFIGS[4]
    ranks = [48] * 3 + [32] * 6 + [16] * 6
    s = hm_inputs.hss_random_ranked(cfg.n, cfg.levels, ranks, cid=51)
    X = hm_inputs.rhs(cfg.n, 32, cid=51)
    g = [dev(a) for a in (s.D, s.U, s.V, s.R, s.W, s.B)]
    Y = hm.hss_matvec_ranked(cfg.n, cfg.levels, cfg.leaf, ranks, *g, dev(X))
    torch.cuda.synchronize()
    Yr = oracle.hss_matvec_ranked(cfg.n, cfg.levels, ranks, s.D, s.U, s.V, s.R, s.W, s.B, X)
    assert relerr(Y.cpu().numpy(), Yr) <= TOL


def test_hss_ranked_errors(hm):
    x = torch.zeros(1024, 1, dtype=torch.float64, device="cuda")
    with pytest.raises(hm.HmError):
        hm.hss_matvec_ranked(1024, 4, 64, [3, 5, 65, 8], x, x, x, x, x, x, x)
    big = torch.zeros(1024 * 64, dtype=torch.float64, device="cuda")
    with pytest.raises(hm.HmError):  # op must be 0 or 1
        hm.hss_matvec_ranked(1024, 4, 64, [3, 5, 7, 8], big, big, big, big, big, big, x, op=2)


# ---------------------------------------------------------- per-node ranks --

def node_ranks_of(p, fn):
    return [int(fn(l, i)) for l in range(1, p + 1) for i in range(1 << l)]


NODE_CASES = [
    # n, levels, per-node rank function (level, index), nrhs
    (1024, 4, lambda l, i: 2 + (3 * i + l) % 7, 1),
    (4096, 6, lambda l, i: 8 + 8 * ((i + l) % 2), 8),                  # 8 / 16 alternating: tuned paths at K_l = 16
    (8192, 7, lambda l, i: (5 * i + 3 * l) % 11, 3),                   # rank-0 nodes
    (1 << 15, 8, lambda l, i: 32 if (i % 4 == 0) else 16 + (i % 3), 32),
    (4096, 6, lambda l, i: 4 * l, 2),                                  # equal within levels: the per-level path
]


@pytest.mark.parametrize("op", [0, 1])
@pytest.mark.parametrize("n,p,fn,m", NODE_CASES)
def test_hss_noderanked_vs_oracle(hm, n, p, fn, m, op):
    kn = node_ranks_of(p, fn)
    s = hm_inputs.hss_random_noderanked(n, p, kn, cid=52)
    X = hm_inputs.rhs(n, m, cid=52)
    g = [dev(a) if a.size else torch.zeros(1, dtype=torch.float64, device="cuda:0")
         for a in (s.D, s.U, s.V, s.R, s.W, s.B)]
    Y = hm.hss_matvec_noderanked(n, p, n >> p, kn, *g, dev(X), op=op)
    torch.cuda.synchronize()
    Yr = oracle.hss_matvec_noderanked(n, p, kn, s.D, s.U, s.V, s.R, s.W, s.B, X, trans=bool(op))
    assert relerr(Y.cpu().numpy(), Yr) <= TOL


def test_hss_noderanked_config4_tree(hm):
    """The config-4 tree (n = 2^22, leaf 128, 15 levels) with per-node ranks 24..32, nrhs 32."""
    cfg = hm_inputs.CONFIGS[4]
    kn = node_ranks_of(cfg.levels, lambda l, i: 24 + (7 * i + l) % 9)
    s = hm_inputs.hss_random_noderanked(cfg.n, cfg.levels, kn, cid=53)
    X = hm_inputs.rhs(cfg.n, 32, cid=53)
    g = [dev(a) for a in (s.D, s.U, s.V, s.R, s.W, s.B)]
    Y = hm.hss_matvec_noderanked(cfg.n, cfg.levels, cfg.leaf, kn, *g, dev(X))
    torch.cuda.synchronize()
    Yr = oracle.hss_matvec_noderanked(cfg.n, cfg.levels, kn, s.D, s.U, s.V, s.R, s.W, s.B, X)
    assert relerr(Y.cpu().numpy(), Yr) <= TOL


@pytest.mark.parametrize("op", [0, 1])
def test_hss_ranked_dmma_levels_ran(hm, op):
    """Per-level ranks that are multiples of 8 run the DMMA level kernels
    (hss_up_ranked_mma / hss_down_ranked_mma, hm_tree.cuh); a level of rank 4 next to
    them keeps the CUDA-core kernels. Every row against the oracle, A and A^T."""
    n, p, m = 1 << 14, 8, 12
    ranks = [24, 16, 16, 8, 4, 8, 16, 24]
    s = hm_inputs.hss_random_ranked(n, p, ranks, cid=52)
    X = hm_inputs.rhs(n, m, cid=52)
    g = [dev(a) for a in (s.D, s.U, s.V, s.R, s.W, s.B)]
    hm.hm_profile_collect()
    hm.hm_profile_enable(True)
    try:
        Y = hm.hss_matvec_ranked(n, p, n >> p, ranks, *g, dev(X), op=op)
        torch.cuda.synchronize()
    finally:
        hm.hm_profile_enable(False)
    names = {t[0] for t in hm.hm_profile_collect()}
    assert {"hss_up_ranked_mma<nt2>", "hss_down_ranked_mma<nt2>", "hss_down_ranked"} <= names, names
    Yr = oracle.hss_matvec_ranked(n, p, ranks, s.D, s.U, s.V, s.R, s.W, s.B, X, trans=bool(op))
    assert relerr(Y.cpu().numpy(), Yr) <= TOL


@pytest.mark.parametrize("op", [0, 1])
def test_hss_ranked_sweep_small_levels(hm, op):
    """The bench sweep's per-level tree (n = 2^20, leaf 128, 13 levels, ranks 32/24/16,
    nrhs 16): the levels with < 2048 nodes of both sweeps run in one cooperative launch
    (hss_ranked_sweep), the bigger ones one DMMA launch each. Every row, A and A^T."""
    n, p, m = 1 << 20, 13, 16
    ranks = [32] * 4 + [24] * 4 + [16] * 5
    s = hm_inputs.hss_random_ranked(n, p, ranks, cid=53)
    X = hm_inputs.rhs(n, m, cid=53)
    g = [dev(a) for a in (s.D, s.U, s.V, s.R, s.W, s.B)]
    hm.hm_profile_collect()
    hm.hm_profile_enable(True)
    try:
        Y = hm.hss_matvec_ranked(n, p, n >> p, ranks, *g, dev(X), op=op)
        torch.cuda.synchronize()
    finally:
        hm.hm_profile_enable(False)
    names = [t[0] for t in hm.hm_profile_collect()]
    assert names.count("hss_ranked_sweep<nt2>") == 1, names
    assert "hss_up_ranked_mma<nt2>" in names and "hss_down_ranked_mma<nt2>" in names, names
    Yr = oracle.hss_matvec_ranked(n, p, ranks, s.D, s.U, s.V, s.R, s.W, s.B, X, trans=bool(op))
    assert relerr(Y.cpu().numpy(), Yr) <= TOL
