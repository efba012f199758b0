"""Host-side arithmetic of bench.py (no GPU): the algorithmic byte / flop counts of
SURVEY §8(d) and config 4's attainable time of DESIGN.md §11."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_step_bytes_match_the_survey_counts():
    c5, c4 = bench.C5, bench.C4
    # config 5: n b + 2 p n k + 2 n m doubles; config 4: n b + 2 n k + 6 (2^p) k^2 (approx.) + 2 n m
    assert bench.hodlr_bytes(c5.n, c5.leaf, c5.levels, c5.k, 1) == 8 * (c5.n * 256 + 2 * 16 * c5.n + 2 * c5.n)
    assert abs(bench.step_bytes() / 1e9 - 49.12) < 0.01


def test_config4_attainable_time():
    """leaf pass 7.8 GB / 42.9 GF at 5.5 flop/B on the measured ridge
    (31.6 TF/s, 1.36 ms) + Step 1 2.41 GB at the read stream (0.34 ms) + the tree
    levels 3.76 GB at the 6523 GB/s copy figure (0.58 ms) = 2.27 ms."""
    c4 = bench.C4
    ms = bench.hss_attainable_ms(c4.n, c4.leaf, c4.levels, c4.k, bench.M4, 6523.3)
    assert abs(ms - 2.27) < 0.01, ms
    # a faster copy figure can only lower it; the naive roofline is below it
    assert bench.hss_attainable_ms(c4.n, c4.leaf, c4.levels, c4.k, bench.M4, 7000.0) < ms
    naive = max(bench.hss_bytes(c4.n, c4.leaf, c4.levels, c4.k, 32) / 6523.3e9,
                bench.hss_flops(c4.n, c4.leaf, c4.levels, c4.k, 32) / 37.0e12) * 1e3
    assert naive < ms
