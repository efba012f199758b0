"""hm_inputs (the seeded generators serving both sides): the OpenMP host fill of
the config-5 leaf blocks gives the same bits as the numpy formula, and the
closed form's defining entries (reading G11)."""
import numpy as np

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
