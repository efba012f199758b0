"""Multi-GPU path on ONE GPU.

1. Split-phase calls: every rank's libhm calls run in this process, one rank
   after the other (no rank waits on another), and the allgather is a plain
   concatenation of the ranks' send buffers. The distributed product (SURVEY
   §8(e)) is checked against the CPU oracle and the single-GPU product, for
   both HODLR schedules (leaf pass overlapped with the exchange + top-level
   epilogue, and the fused leaf pass).
2. One-call products with libhm's NCCL communicator at P = 1 (this pool has one
   GPU per box): hodlr_matvec_dist / hss_matvec_dist / hm_comm_allgather
   through a real ncclComm, against the oracle and the single-GPU product.
   A two-process run needs two GPUs (NCCL rejects two ranks on one device).
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
        Yl = torch.empty_like(Xl)
        hd.hodlr_matvec_dist_local(n, p, b, ranks, P, r, Dl, Ul, Vl, Xl, Yl, wss[r])
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
    (1 << 16, 256, 8, 4, 1, 8),        # overlapped schedule (leaf pass before the exchange, top epilogue)
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
    (8192, 64, 7, 16, 1, 4),           # m = 1 (one masked DMMA column tile)
    (4096, 64, 6, 5, 3, 2),            # generic kernels
    (2048, 64, 5, 16, 2, 32),          # one leaf per rank
    (1024, 64, 4, 16, 4, 8),           # subtree of depth 1
    (1 << 20, 64, 14, 32, 1, 2),       # m = 1 on deep subtrees (depth 13, 12): the DMMA kernels on one masked tile
    (1 << 20, 64, 14, 16, 1, 4),
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


def test_overlap_schedule_selected(hm):
    """The emulated config-5 run above takes the overlapped schedule: _local launches the
    leaf pass, _end the top-level epilogue (the one-call product runs the same)."""
    from paper_1909_07909_b200 import dist as hd
    n, p, b, P, r = 1 << 17, 9, 256, 8, 3
    h = hm_inputs.hodlr_inverse_laplacian(n, p, xp=torch, device="cuda:0")
    Dl, Ul, Vl = hd.hodlr_shard(n, p, b, h.ranks, h.D, h.U, h.V, P, r)
    Xl = torch.ones(n // P, 1, dtype=torch.float64, device="cuda:0")
    Yl = torch.empty_like(Xl)
    wsb, sd = hd.hodlr_dist_sizes(n, p, b, h.ranks, 1, P, r)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda:0")
    gathered = torch.zeros(P * sd, dtype=torch.float64, device="cuda:0")
    hm.hm_profile_collect()
    hm.hm_profile_enable(True)
    hd.hodlr_matvec_dist_local(n, p, b, h.ranks, P, r, Dl, Ul, Vl, Xl, Yl, ws)
    hd.hodlr_matvec_dist_end(n, p, b, h.ranks, P, r, Dl, Ul, Xl, gathered, Yl, ws)
    torch.cuda.synchronize()
    hm.hm_profile_enable(False)
    tr = hm.hm_profile_collect()
    calls = {}
    for name, call, _ in tr:
        calls.setdefault(call, []).append(name)
    assert any(n_.startswith("leaf_gemv") for n_ in calls[0]), calls
    assert "dist_top_epilogue" in calls[1] and not any(n_.startswith("leaf") for n_ in calls[1]), calls


# ------------------------------------------------- one call, NCCL inside (P = 1) --

@pytest.fixture(scope="module")
def comm(hm):
    from paper_1909_07909_b200 import dist as hd
    c = hd.Comm(1, 0, hd.unique_id())
    yield c
    c.close()


def test_comm_allgather_p1(comm):
    x = torch.arange(10, dtype=torch.float64, device="cuda:0")
    y = comm.allgather(x)
    torch.cuda.synchronize()
    assert torch.equal(x, y)


@pytest.mark.parametrize("n,b,p,k,m", [(1 << 16, 256, 8, 16, 8), (1 << 17, 256, 9, 1, 1), (4096, 64, 6, 8, 3)])
def test_hodlr_matvec_dist_nccl_p1(hm, comm, n, b, p, k, m):
    from paper_1909_07909_b200 import dist as hd
    h = hm_inputs.hodlr_random(n, p, [k] * p, cid=23)
    X = hm_inputs.rhs(n, m, cid=23)
    D, U, V, Xd = dev(h.D), dev(h.U), dev(h.V), dev(X)
    s = torch.cuda.Stream()
    Yd = hd.hodlr_matvec_dist(comm, n, p, b, h.ranks, D, U, V, Xd, stream=s)
    s.synchronize()
    Yr = oracle.hodlr_matvec(n, p, h.ranks, h.D, h.U, h.V, X)
    assert relerr(Yd.cpu().numpy(), Yr) <= TOL
    Y1 = hm.hodlr_matvec(n, p, b, h.ranks, D, U, V, Xd)
    torch.cuda.synchronize()
    assert torch.equal(Yd, Y1)


@pytest.mark.parametrize("n,b,p,k,m", [(1 << 15, 128, 8, 32, 32), (8192, 64, 7, 16, 1), (4096, 64, 6, 5, 3)])
def test_hss_matvec_dist_nccl_p1(hm, comm, n, b, p, k, m):
    from paper_1909_07909_b200 import dist as hd
    s = hm_inputs.hss_random(n, p, k, cid=24)
    X = hm_inputs.rhs(n, m, cid=24)
    g = {a: dev(getattr(s, a)) for a in ("D", "U", "V", "R", "W", "B")}
    sh = {kk: v.contiguous() for kk, v in hd.hss_shard(n, p, b, k, g["D"], g["U"], g["V"], g["R"], g["W"], g["B"],
                                                      1, 0).items()}
    Xd = dev(X)
    Yd = hd.hss_matvec_dist(comm, n, p, b, k, sh, Xd)
    torch.cuda.synchronize()
    Yr = oracle.hss_matvec(n, p, k, s.D, s.U, s.V, s.R, s.W, s.B, X)
    assert relerr(Yd.cpu().numpy(), Yr) <= TOL
    Y1 = hm.hss_matvec(n, p, b, k, g["D"], g["U"], g["V"], g["R"], g["W"], g["B"], Xd)
    torch.cuda.synchronize()
    assert relerr(Yd.cpu().numpy(), Y1.cpu().numpy()) <= 1e-14  # the single-GPU call may take hss_small


def test_config5_dist_nccl_p1(hm, comm):
    """Config 5 at full size through the one-call product and the real communicator."""
    from paper_1909_07909_b200 import dist as hd
    cfg = hm_inputs.CONFIGS[5]
    h = hm_inputs.hodlr_inverse_laplacian(cfg.n, cfg.levels, xp=torch, device="cuda:0")
    X = hm_inputs.rhs(cfg.n, 1, cid=5)
    Yd = hd.hodlr_matvec_dist(comm, cfg.n, cfg.levels, cfg.leaf, h.ranks, h.D, h.U, h.V, dev(X))
    torch.cuda.synchronize()
    assert relerr(Yd.cpu().numpy(), oracle.laplacian_inverse_apply(X)) <= TOL


def test_c_dist_example_on_gpu(hm, tmp_path):
    """examples/hm_dist_example.c: plain C, one process per GPU (this box: P = 1), the
    communicator id through a pipe, hodlr_matvec_dist + hss_matvec_dist vs the closed form."""
    import subprocess
    from test_abi import _build_c_example
    exe = _build_c_example(tmp_path, "hm_dist_example")
    ngpu = torch.cuda.device_count()
    P = 1 << (ngpu.bit_length() - 1)
    out = subprocess.run([exe, str(P)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "all ranks OK" in out.stdout


def test_trace_timeline_across_streams(hm, comm):
    """hm_profile_timeline puts the exchange (communicator stream) and the caller's
    kernels on one device timeline: starts are measured from the first record, and
    a kernel queued behind the exchange on the same caller stream starts after it."""
    from paper_1909_07909_b200 import dist as hd
    n, p, b, k, m = 1 << 16, 8, 256, 16, 8
    h = hm_inputs.hodlr_random(n, p, [k] * p, cid=25)
    D, U, V, Xd = dev(h.D), dev(h.U), dev(h.V), dev(hm_inputs.rhs(n, m, cid=25))
    x = torch.arange(1 << 20, dtype=torch.float64, device="cuda:0")
    hm.hm_profile_collect()
    hm.hm_profile_enable(True)
    hm.hodlr_matvec(n, p, b, h.ranks, D, U, V, Xd)
    y = comm.allgather(x)                      # caller stream waits for the exchange
    hm.hodlr_matvec(n, p, b, h.ranks, D, U, V, Xd)
    torch.cuda.synchronize()
    hm.hm_profile_enable(False)
    tr = hm.hm_profile_timeline()
    assert torch.equal(x, y)
    assert tr[0][2] == 0.0
    names = [t[0] for t in tr]
    ix = names.index("nccl_allgather")
    _, _, t_ex, ms_ex = tr[ix]
    first = [t for t in tr[:ix]]
    after = [t for t in tr[ix + 1:]]
    assert first and after
    eps = 2e-3  # ms: event resolution
    assert t_ex + eps >= first[-1][2] + first[-1][3]           # ordered after the caller's work
    assert all(t[2] + eps >= t_ex + ms_ex for t in after)      # the next call waited for it
    for a, c in zip(tr[:ix - 1], tr[1:ix]):                     # one stream: records do not overlap
        assert c[2] + eps >= a[2] + a[3]
