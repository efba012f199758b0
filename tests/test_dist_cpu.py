"""Multi-process (gloo, CPU) checks of the distributed path's host logic.

World sizes 2 and 4, one process per rank, rendezvous on 127.0.0.1. Each rank
shards the generators with paper_1909_07909_b200.dist (the same helpers the GPU
path uses), sizes its exchange block with the library's host-only
hm_*_dist_sizes, exchanges through dist.allgather (gloo here, NCCL on GPUs),
and finishes with a numpy emulation of the _begin/_end phases (the partition
arithmetic of include/hm.h "multi-GPU"). The assembled Y must equal the CPU
oracle. No GPU is used.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def allgather(send, gathered):
    """gathered[P * len(send)] <- concat over ranks of send, rank order (gloo)."""
    if send.numel():
        dist.all_gather_into_tensor(gathered, send)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


# ------------------------------------------------------ numpy phase emulation --

def hodlr_rank(n, p, b, ranks, D, U, V, X, P, r, hd, oracle):
    q = P.bit_length() - 1
    nl = n // P
    m = X.shape[1]
    Dl, Ul, Vl = hd.hodlr_shard(n, p, b, ranks, D, U, V, P, r)
    Xl = X[r * nl:(r + 1) * nl]
    _, sd = hd.hodlr_dist_sizes(n, p, b, ranks, m, P, r)  # host-only library call
    # _begin: partial t_l = V_l(I_r)^T X(I_r), l = 1..q, packed
    send, off = [], 0
    for l in range(1, p + 1):
        k = ranks[l - 1]
        if l <= q:
            send.append((Vl[off:off + nl * k].reshape(nl, k).T @ Xl).ravel())
        off += nl * k
    send = np.concatenate(send) if send else np.zeros(0)
    assert send.size == sd
    gathered = torch.empty(P * sd, dtype=torch.float64)
    allgather(torch.from_numpy(send), gathered)
    gathered = gathered.numpy().reshape(P, sd)
    # _end: subtree product (levels q+1..p on the local rows) + top terms
    sub_ranks = list(ranks[q:])
    Uoff = sum(nl * ranks[l - 1] for l in range(1, q + 1))
    Yl = oracle.hodlr_matvec(nl, p - q, sub_ranks if p > q else [], Dl, Ul[Uoff:], Vl[Uoff:], Xl)
    off, toff = 0, 0
    for l in range(1, q + 1):
        k = ranks[l - 1]
        a = r >> (q - l)
        span = 1 << (q - l)
        t = sum(gathered[rr, toff:toff + k * m] for rr in range((a ^ 1) * span, ((a ^ 1) + 1) * span))
        Yl = Yl + Ul[off:off + nl * k].reshape(nl, k) @ t.reshape(k, m)
        off += nl * k
        toff += k * m
    return Yl


def hss_up(xleaf, W, pl, k, m):
    """Upsweep of a depth-pl subtree from its leaf x blocks; heap layout."""
    xs = {pl: [xleaf[i] for i in range(1 << pl)]}
    Wn = W.reshape(-1, 2 * k, k)
    for l in range(pl - 1, 0, -1):
        xs[l] = [Wn[(1 << l) - 2 + i].T @ np.vstack([xs[l + 1][2 * i], xs[l + 1][2 * i + 1]])
                 for i in range(1 << l)]
    return xs


def hss_down(xs, B, R, pl, k, yroot=None, Rroot=None):
    Bn, Rn = B.reshape(-1, 2, k, k), R.reshape(-1, 2 * k, k)
    ys = {}
    for l in range(1, pl + 1):
        ys[l] = []
        for j in range(1 << l):
            qq, w = j >> 1, j & 1
            y = Bn[(1 << (l - 1)) - 1 + qq, w] @ xs[l][j ^ 1]
            if l >= 2:
                y = y + Rn[(1 << (l - 1)) - 2 + qq][w * k:(w + 1) * k] @ ys[l - 1][qq]
            elif Rroot is not None:
                y = y + Rroot.reshape(2 * k, k)[w * k:(w + 1) * k] @ yroot
            ys[l].append(y)
    return ys


def hss_rank(n, p, b, k, s, X, P, r, hd):
    q = P.bit_length() - 1
    nl, pl, m = n // P, p - q, X.shape[1]
    sh = hd.hss_shard(n, p, b, k, s.D, s.U, s.V, s.R, s.W, s.B, P, r)
    Xl = X[r * nl:(r + 1) * nl]
    _, sd = hd.hss_dist_sizes(n, p, b, k, m, P, r)
    Ul, Vl = sh["U"].reshape(nl, k), sh["V"].reshape(nl, k)
    xleaf = [Vl[i * b:(i + 1) * b].T @ Xl[i * b:(i + 1) * b] for i in range(1 << pl)]
    xs = hss_up(np.array(xleaf), sh["W_sub"], pl, k, m)
    xroot = xleaf[0] if pl == 0 else sh["W_root"].reshape(2 * k, k).T @ np.vstack([xs[1][0], xs[1][1]])
    assert xroot.size == sd
    gathered = torch.empty(P * sd, dtype=torch.float64)
    allgather(torch.from_numpy(np.ascontiguousarray(xroot).ravel()), gathered)
    xq = gathered.numpy().reshape(P, k, m)
    # replicated top tree (levels 1..q)
    txs = hss_up(xq, sh["W_top"], q, k, m)
    tys = hss_down(txs, sh["B_top"], sh["R_top"], q, k)
    yroot = tys[q][r]
    if pl >= 1:
        ys = hss_down(xs, sh["B_sub"], sh["R_sub"], pl, k, yroot=yroot, Rroot=sh["R_root"])
        yleaf = ys[pl]
    else:
        yleaf = [yroot]
    Dl = sh["D"].reshape(-1, b, b)
    return np.vstack([Ul[i * b:(i + 1) * b] @ yleaf[i] + Dl[i] @ Xl[i * b:(i + 1) * b] for i in range(1 << pl)])


def _worker(rank, world, port, case, outdir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import hm_inputs
    import oracle
    from paper_1909_07909_b200 import dist as hd
    kind, n, p, b, k, m = case
    if kind == "hodlr":
        h = hm_inputs.hodlr_random(n, p, [k] * p, cid=31)
        X = hm_inputs.rhs(n, m, cid=31)
        Yl = hodlr_rank(n, p, b, [k] * p, h.D, h.U, h.V, X, world, rank, hd, oracle)
        Yref = oracle.hodlr_matvec(n, p, h.ranks, h.D, h.U, h.V, X)
    else:
        s = hm_inputs.hss_random(n, p, k, cid=32)
        X = hm_inputs.rhs(n, m, cid=32)
        Yl = hss_rank(n, p, b, k, s, X, world, rank, hd)
        Yref = oracle.hss_matvec(n, p, k, s.D, s.U, s.V, s.R, s.W, s.B, X)
    parts = [torch.empty(Yl.size, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(Yl).ravel()))
    if rank == 0:
        Y = np.concatenate([t.numpy() for t in parts]).reshape(n, m)
        err = np.linalg.norm(Y - Yref) / np.linalg.norm(Yref)
        with open(os.path.join(outdir, "err.txt"), "w") as f:
            f.write(repr(float(err)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [
    (2, ("hodlr", 4096, 6, 64, 8, 3)),
    (4, ("hodlr", 4096, 6, 64, 8, 2)),
    (4, ("hodlr", 1024, 2, 256, 4, 1)),   # one leaf per rank
    (2, ("hss", 4096, 6, 64, 8, 3)),
    (4, ("hss", 2048, 5, 64, 4, 2)),
    (4, ("hss", 1024, 2, 256, 4, 2)),     # one leaf per rank
])
def test_dist_gloo(tmp_path, world, case):
    from paper_1909_07909_b200 import build
    build.build()
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, case, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    err = float(open(tmp_path / "err.txt").read())
    assert err < 1e-13, err


def _id_worker(rank, world, port, outdir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1909_07909_b200 import dist as hd
    uid = hd.broadcast_unique_id()
    with open(os.path.join(outdir, f"id{rank}.bin"), "wb") as f:
        f.write(uid)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_comm_unique_id_broadcast_gloo(tmp_path, world):
    """Comm.from_group's out-of-band step: rank 0's libhm (NCCL) unique id reaches every
    rank byte for byte (the host half of hm_comm_init; the NCCL half needs GPUs)."""
    from paper_1909_07909_b200 import build
    build.build()
    mp.start_processes(_id_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    ids = [open(tmp_path / f"id{r}.bin", "rb").read() for r in range(world)]
    assert len(ids[0]) == 128 and any(ids[0]) and all(i == ids[0] for i in ids)
