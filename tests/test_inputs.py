"""hm_inputs (the seeded generators serving both sides): the OpenMP host fill of
the config-5 leaf blocks gives the same bits as the numpy formula, and the
closed form's defining entries (reading G11)."""
import numpy as np
import pytest

import hm_inputs


def test_fill_matches_numpy_formula():
    n, p = 1 << 14, 6
    fast = hm_inputs.inverse_laplacian_leaf_blocks(n, p)                      # contiguous: fill.c
    slow = hm_inputs.inverse_laplacian_leaf_blocks(n, p, leaves=list(range(1 << p)))  # numpy path
    assert np.array_equal(fast, slow)
    part = hm_inputs.inverse_laplacian_leaf_blocks(n, p, leaves=range(7, 19))
    assert np.array_equal(part, slow[7 * 256 * 256:19 * 256 * 256])


def test_fill_entries_closed_form():
    n, p = 1000, 3  # leaf 125
    D = hm_inputs.inverse_laplacian_leaf_blocks(n, p).reshape(8, 125, 125)
    for L, r, c in ((0, 0, 0), (3, 10, 100), (7, 124, 0)):
        i, j = L * 125 + r + 1, L * 125 + c + 1
        assert D[L, r, c] == min(i, j) * (n + 1 - max(i, j)) / (n + 1)


def test_device_hss_shard_matches_global_sharding():
    """bench.py's shard-local fill: every rank's shard (drawn alone) equals the shard of
    the global matrix (the P = 1 draw) cut by paper_1909_07909_b200.dist.hss_shard."""
    torch = pytest.importorskip("torch")
    from paper_1909_07909_b200 import dist as hd
    n, p, k = 4096, 5, 8
    full = hm_inputs.device_hss_shard(n, p, k, 7, "cpu", 1, 0, block=4)
    g = {"D": full["D"], "U": full["U"], "V": full["V"], "R": full["R_sub"], "W": full["W_sub"], "B": full["B_sub"]}
    for P in (2, 4, 32):
        for r in range(P):
            a = hm_inputs.device_hss_shard(n, p, k, 7, "cpu", P, r, block=4)
            b = hd.hss_shard(n, p, n >> p, k, g["D"], g["U"], g["V"], g["R"], g["W"], g["B"], P, r)
            for key in a:
                assert torch.equal(a[key], b[key].contiguous()), (P, r, key)


def test_inverse_laplacian_factor_rows():
    U, V = hm_inputs.inverse_laplacian_factors(1 << 10, 4)
    Us, Vs = hm_inputs.inverse_laplacian_factors(1 << 10, 4, rows=(256, 512))
    assert np.array_equal(Us.reshape(4, 256), U.reshape(4, 1024)[:, 256:512])
    assert np.array_equal(Vs.reshape(4, 256), V.reshape(4, 1024)[:, 256:512])
