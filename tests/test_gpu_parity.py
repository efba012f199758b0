"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle, element by element.

Tolerance (BASELINE.json north_star): ||Y_gpu - Y_ref||_F / ||Y_ref||_F <= 1e-12 in fp64.
Inputs: seeded, from hm_inputs; the same bytes feed both sides.
Small cases run the full oracle; configs 3 and 4 at full size are compared with
the full oracle on every row in test_gpu_fullsize.py; config 5 (n = 2^24) here on
every row against the closed-form oracle, plus sampled leaves through the HODLR
oracle, and closed forms that hold at any size.
"""
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


def gpu_hodlr(hm, h, X):
    Y = hm.hodlr_matvec(h.n, h.levels, h.leaf, h.ranks, dev(h.D), dev(h.U), dev(h.V), dev(X))
    torch.cuda.synchronize()
    return Y.cpu().numpy()


def gpu_hss(hm, s, X):
    Y = hm.hss_matvec(s.n, s.levels, s.leaf, s.k, dev(s.D), dev(s.U), dev(s.V), dev(s.R), dev(s.W), dev(s.B), dev(X))
    torch.cuda.synchronize()
    return Y.cpu().numpy()


def ref_hodlr(h, X):
    return oracle.hodlr_matvec(h.n, h.levels, h.ranks, h.D, h.U, h.V, X)


def ref_hss(s, X):
    return oracle.hss_matvec(s.n, s.levels, s.k, s.D, s.U, s.V, s.R, s.W, s.B, X)


def tridiag_residual(Y, X):
    TY = 2 * Y
    TY[1:] -= Y[:-1]
    TY[:-1] -= Y[1:]
    normT = 2 + 2 * np.cos(np.pi / (Y.shape[0] + 1))
    return np.linalg.norm(TY - X) / (normT * np.linalg.norm(Y) + np.linalg.norm(X))


# ------------------------------------------------------------ small, full oracle --

HODLR_CASES = [
    # n, leaf, levels, k, nrhs
    (1024, 64, 4, 8, 1),        # BASELINE config 1 in full
    (256, 16, 4, 3, 3),
    (512, 64, 3, 5, 17),        # nrhs > one column chunk, ragged chunk
    (384, 48, 3, 4, 2),         # non-power-of-two leaf
    (100, 100, 0, 0, 4),        # depth 0: Y = D X
    (2048, 32, 6, 0, 2),        # every rank 0: block diagonal
    (8192, 256, 5, 64, 8),      # maximum rank
    (65536, 256, 8, 16, 1),     # many row tiles: partial sums on the top levels
    (65536, 128, 9, 4, 64),
    (4096, 1, 12, 1, 1),        # leaf size 1 (Fig. 1's n_min = 1)
    (65536, 256, 8, 16, 64),    # config-3 shapes (DMMA paths), smaller depth
    (65536, 128, 9, 32, 33),    # DMMA paths, ragged column chunk
    (32768, 64, 9, 16, 2),
    (8192, 256, 5, 16, 8),
    (16384, 64, 8, 2, 1),       # GEMV paths, rank 2
    (32768, 128, 8, 64, 1),     # GEMV paths, rank 64
    (32768, 64, 9, 8, 5),       # small-rank DMMA V^T X (one tile holds every rank column)
    (65536, 256, 8, 8, 64),
    (16384, 128, 7, 2, 9),      # small-rank DMMA, ragged column chunk
    (16384, 64, 8, 1, 2),
    (32768, 128, 8, 32, 32),    # level-parallel pipelined V^T X (vt_lv, m > 16)
    (16384, 64, 8, 16, 17),     # vt_lv, odd m: synchronous X staging, padded columns
    (65536, 256, 8, 16, 48),    # vt_lv, 3 work items per warp
    (16384, 256, 6, 16, 100),   # nrhs > 64: several column chunks of every kernel
    (8192, 64, 7, 32, 129),
    (4096, 128, 5, 8, 200),
]


@pytest.mark.parametrize("n,leaf,levels,k,m", HODLR_CASES)
def test_hodlr_vs_oracle(hm, n, leaf, levels, k, m):
    h = hm_inputs.hodlr_random(n, levels, [k] * levels, cid=11)
    X = hm_inputs.rhs(n, m, cid=11)
    Yg = gpu_hodlr(hm, h, X)
    Yr = ref_hodlr(h, X)
    assert relerr(Yg, Yr) <= TOL


HSS_CASES = [
    (4096, 64, 6, 16, 16),      # BASELINE config 2 in full
    (256, 16, 4, 3, 3),
    (384, 48, 3, 4, 2),
    (100, 100, 0, 4, 2),        # depth 0
    (64, 32, 1, 4, 5),          # p = 1: cores at the root only, no translations
    (2048, 32, 6, 0, 2),        # k = 0: block diagonal (G17)
    (8192, 64, 7, 64, 3),       # maximum rank
    (32768, 128, 8, 32, 32),    # config-4 shapes at a smaller depth
    (4096, 64, 6, 16, 33),      # ragged column chunk
    (8192, 64, 7, 16, 1),       # GEMV paths
    (16384, 256, 6, 32, 8),
    (16384, 128, 7, 64, 5),
    (2048, 128, 4, 16, 2),
    (16384, 128, 7, 32, 100),   # nrhs > 64: several column chunks of every kernel
    (8192, 64, 7, 16, 129),
]


@pytest.mark.parametrize("n,leaf,levels,k,m", HSS_CASES)
def test_hss_vs_oracle(hm, n, leaf, levels, k, m):
    s = hm_inputs.hss_random(n, levels, k, cid=12)
    X = hm_inputs.rhs(n, m, cid=12)
    Yg = gpu_hss(hm, s, X)
    Yr = ref_hss(s, X)
    assert relerr(Yg, Yr) <= TOL


@pytest.mark.parametrize("level", [1, 2, 5, 8])
def test_hodlr_level_isolation(hm, level):
    """G14: D = 0, only level `level` non-zero — a level-local error cannot hide."""
    n, b, p, k, m = 1 << 16, 256, 8, 16, 8
    h = hm_inputs.hodlr_random(n, p, [k] * p, cid=13)
    h.D[:] = 0
    for l in range(1, p + 1):
        if l != level:
            h.U[h.level_slice(l)] = 0
    X = hm_inputs.rhs(n, m, cid=13)
    Yr = ref_hodlr(h, X)
    assert np.linalg.norm(Yr) > 0
    assert relerr(gpu_hodlr(hm, h, X), Yr) <= TOL


@pytest.mark.parametrize("level", [1, 3, 6])
def test_hss_level_isolation(hm, level):
    """D = 0 and cores zero except the level-`level` sibling pairs."""
    n, b, p, k, m = 8192, 64, 7, 8, 4
    s = hm_inputs.hss_random(n, p, k, cid=14)
    s.D[:] = 0
    B = s.B.reshape(-1, 2, k, k)
    lo, hi = (1 << (level - 1)) - 1, (1 << level) - 1   # parents at level-1 hold level-`level` cores
    B[:lo] = 0
    B[hi:] = 0
    X = hm_inputs.rhs(n, m, cid=14)
    Yr = ref_hss(s, X)
    assert np.linalg.norm(Yr) > 0
    assert relerr(gpu_hss(hm, s, X), Yr) <= TOL


def test_deterministic_and_hostio(hm):
    n, b, p, k, m = 1 << 16, 256, 8, 16, 8
    h = hm_inputs.hodlr_random(n, p, [k] * p, cid=15)
    X = hm_inputs.rhs(n, m, cid=15)
    D, U, V, Xd = dev(h.D), dev(h.U), dev(h.V), dev(X)
    Y1 = hm.hodlr_matvec(n, p, b, h.ranks, D, U, V, Xd)
    Y2 = hm.hodlr_matvec(n, p, b, h.ranks, D, U, V, Xd)
    Xh = torch.from_numpy(X).pin_memory()
    Yh = torch.empty_like(Xh).pin_memory()
    hm.hodlr_matvec_hostio(n, p, b, h.ranks, D, U, V, Xh, Yh)
    torch.cuda.synchronize()
    assert torch.equal(Y1, Y2)
    assert torch.equal(Y1.cpu(), Yh)
    s = hm_inputs.hss_random(8192, 6, 16, cid=15)
    X = hm_inputs.rhs(8192, 4, cid=15)
    args = [dev(a) for a in (s.D, s.U, s.V, s.R, s.W, s.B)]
    Z1 = hm.hss_matvec(8192, 6, s.leaf, 16, *args, dev(X))
    Z2 = hm.hss_matvec(8192, 6, s.leaf, 16, *args, dev(X))
    Xh = torch.from_numpy(X).pin_memory()
    Zh = torch.empty_like(Xh).pin_memory()
    hm.hss_matvec_hostio(8192, 6, s.leaf, 16, *args, Xh, Zh)
    torch.cuda.synchronize()
    assert torch.equal(Z1, Z2) and torch.equal(Z1.cpu(), Zh)


def test_errors_surface(hm):
    x = torch.zeros(1024, 1, dtype=torch.float64, device="cuda")
    with pytest.raises(hm.HmError):
        hm.hodlr_matvec(1000, 2, 256, [4, 4], x, x, x, x)


# ---------------------------------------------------------- closed forms, any size --

def test_inverse_laplacian_hodlr_config3_tree(hm):
    """Config-3 tree (n = 2^20, leaf 256, 12 levels) carrying the exact rank-1 inverse Laplacian."""
    n, p = 1 << 20, 12
    h = hm_inputs.hodlr_inverse_laplacian(n, p)
    X = hm_inputs.rhs(n, 1, cid=5)
    Y = gpu_hodlr(hm, h, X)
    assert relerr(Y, oracle.laplacian_inverse_apply(X)) <= TOL
    assert tridiag_residual(Y, X) <= 1e-14


def test_inverse_laplacian_hss_config4_tree(hm):
    """Config-4 tree (n = 2^22, leaf 128, 15 levels) with the exact rank-2 HSS inverse
    Laplacian: pins every level of the up/coupling/down sweeps at full depth."""
    n, p = 1 << 22, 15
    s = hm_inputs.hss_inverse_laplacian(n, p)
    X = hm_inputs.rhs(n, 1, cid=5)
    Y = gpu_hss(hm, s, X)
    assert relerr(Y, oracle.laplacian_inverse_apply(X)) <= TOL
    assert tridiag_residual(Y, X) <= 1e-14


# --------------------------------------------- full-size configs, sampled leaves --

def sample_leaves(nl, rng, extra=4):
    base = {0, 1, nl // 2 - 1, nl // 2, nl - 1}
    base |= set(int(v) for v in rng.integers(0, nl, size=extra))
    return sorted(base)


def test_config5_full_size(hm):
    """Config 5 (n = 2^24, leaf 256, 16 levels, k = 1): generators filled on the device
    from the closed form (bit-identical to the host formula); every entry of Y against
    the O(n) closed-form oracle, plus tridiag(-1,2,-1) Y = X (G12) and sampled leaves
    through the HODLR oracle."""
    cfg = hm_inputs.CONFIGS[5]
    n, p, b = cfg.n, cfg.levels, cfg.leaf
    hd = hm_inputs.hodlr_inverse_laplacian(n, p, xp=torch, device="cuda:0")
    X = hm_inputs.rhs(n, 1, cid=5)
    Y = hm.hodlr_matvec(n, p, b, hd.ranks, hd.D, hd.U, hd.V, dev(X))
    torch.cuda.synchronize()
    Y = Y.cpu().numpy()
    assert relerr(Y, oracle.laplacian_inverse_apply(X)) <= TOL
    assert tridiag_residual(Y, X) <= 1e-14
    # sampled leaves through the HODLR oracle on host-filled generators (same bits)
    leaves = sample_leaves(cfg.nleaves, np.random.default_rng(5))
    Uh, Vh = hm_inputs.inverse_laplacian_factors(n, p)
    Dsel = hm_inputs.inverse_laplacian_leaf_blocks(n, p, leaves=leaves)
    assert torch.equal(torch.from_numpy(Uh), hd.U.cpu()) and torch.equal(torch.from_numpy(Vh), hd.V.cpu())
    Dsel_dev = torch.cat([hd.D[L * b * b:(L + 1) * b * b] for L in leaves]).cpu().numpy()
    assert np.array_equal(Dsel, Dsel_dev)
    Yr = oracle.hodlr_matvec_leaves(n, p, hd.ranks, Dsel, Uh, Vh, X, leaves)
    Yg = np.concatenate([Y[L * b:(L + 1) * b] for L in leaves])
    assert relerr(Yg, Yr) <= TOL


def test_c_example_on_gpu(hm, tmp_path):
    """examples/hm_matvec_example.c: plain C through the C-ABI on the GPU (A X and A^T X of the
    inverse Laplacian, tridiag(-1,2,-1) residual <= 1e-14)."""
    import subprocess
    from test_abi import _build_c_example
    exe = _build_c_example(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "A^T X: tridiag residual" in out.stdout
