"""Small calls through every kernel family (uniform HODLR / HSS, adjoints,
per-level ranks, small-rank and many-RHS V^T X, ragged general trees), each
checked against the oracle: a quick all-paths check on a GPU box. (Written for
compute-sanitizer; that tool is closed on this pool.)

    python tools/sanitize_cases.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import hm_inputs  # noqa: E402
import oracle  # noqa: E402
import paper_1909_07909_b200 as hm  # noqa: E402
from test_oracle import random_hodlr_general, random_hss_general  # noqa: E402

dev = torch.device("cuda:0")


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def check(name, Y, Yr):
    e = rel(Y.cpu().numpy(), Yr)
    print(f"{name:<44} relerr {e:.2e}")
    assert e <= 1e-12, name


def main():
    # HODLR uniform: GEMV (m=1), DMMA (m=8), small-rank DMMA, vt_lv (m=40), per-level ranks
    for n, p, k, m in ((16384, 6, 16, 1), (16384, 6, 16, 8), (8192, 5, 4, 3), (16384, 6, 16, 40), (8192, 5, 32, 33)):
        h = hm_inputs.hodlr_random(n, p, [k] * p, cid=21)
        X = hm_inputs.rhs(n, m, cid=21)
        Y = hm.hodlr_matvec(n, p, n >> p, h.ranks, t(h.D), t(h.U), t(h.V), t(X))
        check(f"hodlr n={n} p={p} k={k} m={m}", Y, oracle.hodlr_matvec(n, p, h.ranks, h.D, h.U, h.V, X))
        Y = hm.hodlr_matvec_t(n, p, n >> p, h.ranks, t(h.D), t(h.U), t(h.V), t(X))
        check(f"hodlr^T n={n} p={p} k={k} m={m}", Y, oracle.hodlr_matvec_t(n, p, h.ranks, h.D, h.U, h.V, X))
    for ranks, m in (([16, 8, 16, 4, 32], 1), ([16, 32, 8, 16, 16], 8)):
        n, p = 8192, 5
        rng = np.random.default_rng(5)
        c = np.arange(1, (1 << p) + 1, dtype=np.int64) * (n >> p)
        D, U, V = random_hodlr_general(c, p, ranks, rng)
        X = rng.standard_normal((n, m))
        Y = hm.hodlr_matvec(n, p, n >> p, ranks, t(D), t(U), t(V), t(X))
        check(f"hodlr per-level ranks {ranks} m={m}", Y, oracle.hodlr_matvec(n, p, ranks, D, U, V, X))
    # HSS uniform: small-tree one-launch path, level kernels (DMMA / GEMV)
    for n, p, k, m in ((4096, 6, 16, 16), (65536, 9, 32, 32), (65536, 9, 32, 1), (32768, 8, 16, 8)):
        s = hm_inputs.hss_random(n, p, k, cid=22)
        X = hm_inputs.rhs(n, m, cid=22)
        g = [t(a) for a in (s.D, s.U, s.V, s.R, s.W, s.B)]
        Y = hm.hss_matvec(n, p, n >> p, k, *g, t(X))
        check(f"hss n={n} p={p} k={k} m={m}", Y, oracle.hss_matvec(n, p, k, s.D, s.U, s.V, s.R, s.W, s.B, X))
        Y = hm.hss_matvec_t(n, p, n >> p, k, *g, t(X))
        check(f"hss^T n={n} p={p} k={k} m={m}", Y, oracle.hss_matvec_t(n, p, k, s.D, s.U, s.V, s.R, s.W, s.B, X))
    # general (ragged) trees: GEMV / DMMA V^T X, CUDA-core / DMMA leaf pass
    rng = np.random.default_rng(7)
    p = 5
    w = rng.uniform(0.3, 1.7, size=1 << p)
    w[3] = 0.0
    c = np.floor(np.cumsum(w) / w.sum() * 9000).astype(np.int64)
    c[-1] = 9000
    n = 9000
    for ranks, m in (([16] * p, 1), ([16] * p, 8), ([3, 0, 7, 16, 5], 5)):
        D, U, V = random_hodlr_general(c, p, ranks, rng)
        X = rng.standard_normal((n, m))
        for op in (0, 1):
            Y = hm.hodlr_matvec_general(n, p, c, ranks, t(D), t(U), t(V), t(X), op=op)
            f = oracle.hodlr_matvec_t if op else oracle.hodlr_matvec
            check(f"hodlr general ranks {ranks} m={m} op={op}", Y, f(n, p, ranks, D, U, V, X, c=c))
    D, U, V, R, W, B = random_hss_general(c, p, 16, rng)
    X = rng.standard_normal((n, 4))
    Y = hm.hss_matvec_general(n, p, c, 16, *[t(a) for a in (D, U, V, R, W, B)], t(X))
    check("hss general k=16 m=4", Y, oracle.hss_matvec(n, p, 16, D, U, V, R, W, B, X, c=c))
    torch.cuda.synchronize()
    print("sanitize cases: all ok")


if __name__ == "__main__":
    main()
