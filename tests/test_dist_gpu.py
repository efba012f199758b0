"""Multi-GPU path on ONE GPU: every rank's libhm calls run in this process, one
rank after the other (no rank waits on another), and the allgather is a plain
concatenation of the ranks' send buffers. Checks the distributed product
 against the CPU oracle and against the single-GPU product."""
import numpy as np
import pytest

import hm_inputs
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module")
def hm():
    assert torch.cuda.is_available()
    import paper_1909_07909_b200 as hm_
    from paper_1909_07909_b200 import build
    build.build()
    hm_.load()
    return hm_


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda:0")


def relerr(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def emulate_hodlr(hd, n, p, b, ranks, D, U, V, X, P):
    nl = n // P
    shards, sends, wss = [], [], []
    for r in range(P):
        Dl, Ul, Vl = hd.hodlr_shard(n, p, b, ranks, D, U, V, P, r)
        Xl = X[r * nl:(r + 1) * nl].contiguous()
        wsb, sd = hd.hodlr_dist_sizes(n, p, b, ranks, X.shape[1], P, r)
        ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device="cuda:0")
        send = torch.empty(max(sd, 1), dtype=torch.float64, device="cuda:0")[:sd]
        hd.hodlr_matvec_dist_begin(n, p, b, ranks, P, r, Vl, Xl, send, ws)
        shards.append((Dl, Ul, Vl, Xl))
        sends.append(send)
        wss.append(ws)
    gathered = torch.cat(sends)
    Ys = []
    for r in range(P):
        Dl, Ul, Vl, Xl = shards[r]
        hd.hodlr_matvec_dist_local(n, p, b, ranks, P, r, Vl, Xl, wss[r])
        Yl = torch.empty_like(Xl)
        hd.hodlr_matvec_dist_end(n, p, b, ranks, P, r, Dl, Ul, Xl, gathered, Yl, wss[r])
        Ys.append(Yl)
    torch.cuda.synchronize()
    return torch.cat(Ys).cpu().numpy()


def emulate_hss(hd, n, p, b, k, g, X, P):
    nl = n // P
    shards, sends, wss = [], [], []
    for r in range(P):
        sh = hd.hss_shard(n, p, b, k, g["D"], g["U"], g["V"], g["R"], g["W"], g["B"], P, r)
        sh = {kk: v.contiguous() for kk, v in sh.items()}
        Xl = X[r * nl:(r + 1) * nl].contiguous()
        wsb, sd = hd.hss_dist_sizes(n, p, b, k, X.shape[1], P, r)
        ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device="cuda:0")
        send = torch.empty(max(sd, 1), dtype=torch.float64, device="cuda:0")[:sd]
        hd.hss_matvec_dist_begin(n, p, b, k, P, r, sh, Xl, send, ws)
        shards.append((sh, Xl))
        sends.append(send)
        wss.append(ws)
    gathered = torch.cat(sends)
    Ys = []
    for r in range(P):
        sh, Xl = shards[r]
        Yl = torch.empty_like(Xl)
        hd.hss_matvec_dist_end(n, p, b, k, P, r, sh, Xl, gathered, Yl, wss[r])
        Ys.append(Yl)
    torch.cuda.synchronize()
    return torch.cat(Ys).cpu().numpy()


@pytest.mark.parametrize("n,b,p,k,m,P", [
    (1 << 16, 256, 8, 16, 1, 2), (1 << 16, 256, 8, 16, 8, 4), (1 << 16, 256, 8, 16, 8, 8),
    (1 << 16, 256, 8, 16, 8, 1), (1 << 17, 256, 9, 1, 1, 1),   # one rank: the whole tree local
    (1 << 17, 256, 9, 1, 1, 8),        # config-5 shape (k = 1)
    (4096, 64, 6, 8, 3, 4),            # generic kernels
    (2048, 64, 5, 16, 2, 32),          # one leaf per rank (P = 2^p)
    (1 << 16, 128, 9, 32, 33, 2),
    (1 << 16, 256, 8, 16, 64, 4),      # vt_lv on the subtree, top levels as tile partials
])
def test_hodlr_dist_emulated(hm, n, b, p, k, m, P):
    from paper_1909_07909_b200 import dist as hd
    h = hm_inputs.hodlr_random(n, p, [k] * p, cid=21)
    X = hm_inputs.rhs(n, m, cid=21)
    D, U, V, Xd = dev(h.D), dev(h.U), dev(h.V), dev(X)
    Yd = emulate_hodlr(hd, n, p, b, h.ranks, D, U, V, Xd, P)
    Yr = oracle.hodlr_matvec(n, p, h.ranks, h.D, h.U, h.V, X)
    assert relerr(Yd, Yr) <= TOL
    Y1 = hm.hodlr_matvec(n, p, b, h.ranks, D, U, V, Xd).cpu().numpy()
    assert relerr(Yd, Y1) <= 1e-14


@pytest.mark.parametrize("n,b,p,k,m,P", [
    (1 << 15, 128, 8, 32, 32, 2), (1 << 15, 128, 8, 32, 32, 8), (1 << 15, 128, 8, 32, 32, 4),
    (1 << 15, 128, 8, 32, 32, 1), (8192, 64, 7, 16, 1, 1),     # one rank
    (8192, 64, 7, 16, 1, 4),           # m = 1 kernels
    (4096, 64, 6, 5, 3, 2),            # generic kernels
    (2048, 64, 5, 16, 2, 32),          # one leaf per rank
    (1024, 64, 4, 16, 4, 8),           # subtree of depth 1
])
def test_hss_dist_emulated(hm, n, b, p, k, m, P):
    from paper_1909_07909_b200 import dist as hd
    s = hm_inputs.hss_random(n, p, k, cid=22)
    X = hm_inputs.rhs(n, m, cid=22)
    g = {a: dev(getattr(s, a)) for a in ("D", "U", "V", "R", "W", "B")}
    Xd = dev(X)
    Yd = emulate_hss(hd, n, p, b, k, g, Xd, P)
    Yr = oracle.hss_matvec(n, p, k, s.D, s.U, s.V, s.R, s.W, s.B, X)
    assert relerr(Yd, Yr) <= TOL
    Y1 = hm.hss_matvec(n, p, b, k, g["D"], g["U"], g["V"], g["R"], g["W"], g["B"], Xd).cpu().numpy()
    assert relerr(Yd, Y1) <= 1e-14


def test_config5_dist_emulated_8(hm):
    """Config 5 at P = 8 (n = 2^24): distributed result vs the closed form."""
    from paper_1909_07909_b200 import dist as hd
    cfg = hm_inputs.CONFIGS[5]
    n, p, b = cfg.n, cfg.levels, cfg.leaf
    h = hm_inputs.hodlr_inverse_laplacian(n, p, xp=torch, device="cuda:0")
    X = hm_inputs.rhs(n, 1, cid=5)
    Yd = emulate_hodlr(hd, n, p, b, h.ranks, h.D, h.U, h.V, dev(X), 8)
    assert relerr(Yd, oracle.laplacian_inverse_apply(X)) <= TOL
