"""Multi-GPU HODLR / HSS matvec: one process per GPU, P = 2^q ranks.

Rank r owns the rows of the level-q node (q, r) and its whole subtree; the only
exchange is one allgather of small coefficient blocks per product, done INSIDE
libhm by an NCCL communicator (include/hm.h "multi-GPU"):
  HODLR: the rank's partial top-level products V_l(I_r)^T X(I_r), l = 1..q,
         overlapped with the subtree's V^T X and leaf pass;
  HSS:   the x block of node (q, r) (Step 1 up to the subtree root).
This module only marshals: it shards the generators (index arithmetic),
broadcasts the communicator's unique id through torch.distributed (the one
thing the C-ABI leaves to the caller), allocates buffers with torch and calls
hodlr_matvec_dist / hss_matvec_dist. The split-phase calls (*_dist_begin /
_local / _end) are wrapped too: the tests run every rank's kernels on one GPU
with them, the exchange replaced by a concatenation.
"""
from __future__ import annotations

import contextlib
import ctypes
from typing import Sequence

from . import (HM_ERR_INVALID_ARG, HmError, _check, _dev, _ptr, _ranks, _stream, hm_tree, load, make_tree)

HM_COMM_ID_BYTES = 128


class hm_part(ctypes.Structure):
    _fields_ = [("nranks", ctypes.c_int32), ("rank", ctypes.c_int32)]


_sigs_done = False


def _lib():
    global _sigs_done
    lib = load()
    if not _sigs_done:
        P, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        T, PT = ctypes.POINTER(hm_tree), ctypes.POINTER(hm_part)
        sigs = {
            "hm_comm_unique_id": [P],
            "hm_comm_init": [i32, i32, P, ctypes.POINTER(P)],
            "hm_comm_destroy": [P],
            "hm_comm_size": [P, ctypes.POINTER(i32), ctypes.POINTER(i32)],
            "hm_comm_allgather": [P, P, i64, P, P],
            "hm_hodlr_dist_workspace_bytes": [T, P, i32, i32, ctypes.POINTER(sz)],
            "hodlr_matvec_dist": [P, T, P, P, P, P, P, i32, P, P, sz, P],
            "hm_hss_dist_workspace_bytes": [T, i32, i32, i32, ctypes.POINTER(sz)],
            "hss_matvec_dist": [P, T, i32] + [P] * 12 + [i32, P, P, sz, P],
            "hm_hodlr_dist_sizes": [T, P, i32, PT, ctypes.POINTER(sz), ctypes.POINTER(i64)],
            "hodlr_matvec_dist_begin": [T, P, PT, P, P, i32, P, P, sz, P],
            "hodlr_matvec_dist_local": [T, P, PT, P, P, P, P, i32, P, P, sz, P],
            "hodlr_matvec_dist_end": [T, P, PT, P, P, P, i32, P, P, P, sz, P],
            "hm_hss_dist_sizes": [T, i32, i32, PT, ctypes.POINTER(sz), ctypes.POINTER(i64)],
            "hss_matvec_dist_begin": [T, i32, PT, P, P, P, P, i32, P, P, sz, P],
            "hss_matvec_dist_end": [T, i32, PT, P, P, P, P, P, P, P, P, P, i32, P, P, P, sz, P],
        }
        for name, args in sigs.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        _sigs_done = True
    return lib


def _on(stream):
    """Run allocations and the call on the caller's stream (torch's current one if None)."""
    import torch
    return torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()


def _q(P: int) -> int:
    q = P.bit_length() - 1
    if P < 1 or (1 << q) != P:
        raise ValueError(f"the number of ranks ({P}) must be a power of two")
    return q


# ------------------------------------------------------------------ shards --

def hodlr_shard(n: int, levels: int, leaf: int, ranks: Sequence[int], D, U, V, P: int, r: int):
    """Rank r's HODLR generators (include/hm.h "multi-GPU"): its leaves of D and rows
    I_r of every level of U, V (level-major, n/P rows per level). Works on numpy
    arrays or torch tensors (returns views / concatenations)."""
    q = _q(P)
    if q > levels:
        raise ValueError("P > 2^levels")
    nl = n // P
    lpr = (1 << levels) // P
    b2 = leaf * leaf
    D_l = D[r * lpr * b2:(r + 1) * lpr * b2]
    cat = _cat_for(U)
    us, vs, off = [], [], 0
    for l in range(1, levels + 1):
        k = int(ranks[l - 1])
        us.append(U[off + r * nl * k: off + (r + 1) * nl * k])
        vs.append(V[off + r * nl * k: off + (r + 1) * nl * k])
        off += n * k
    return D_l, cat(us), cat(vs)


def hss_shard(n: int, levels: int, leaf: int, k: int, D, U, V, R, W, B, P: int, r: int):
    """Rank r's HSS generators: D, U, V rows I_r; the subtree's W, R (local levels
    1..p-q-1) and B (local levels 0..p-q-1) in heap order relative to node (q, r);
    that node's own W_root, R_root; the replicated top prefixes W_top, R_top
    (levels 1..q-1) and B_top (levels 0..q-1). Returns a dict."""
    q = _q(P)
    if q > levels:
        raise ValueError("P > 2^levels")
    nl = n // P
    lpr = (1 << levels) // P
    b2 = leaf * leaf
    t = 2 * k * k      # one R / W node
    bb = 2 * k * k     # one B node (B12, B21)
    pl = levels - q
    cat = _cat_for(U)
    Wsub, Rsub, Bsub = [], [], []
    for lp in range(1, pl):           # local levels with translations
        g = q + lp
        s0 = (1 << g) - 2 + (r << lp)
        Wsub.append(W[s0 * t:(s0 + (1 << lp)) * t])
        Rsub.append(R[s0 * t:(s0 + (1 << lp)) * t])
    for lp in range(0, pl):           # local levels with cores
        g = q + lp
        s0 = (1 << g) - 1 + (r << lp)
        Bsub.append(B[s0 * bb:(s0 + (1 << lp)) * bb])
    out = {
        "D": D[r * lpr * b2:(r + 1) * lpr * b2],
        "U": U[r * nl * k:(r + 1) * nl * k],
        "V": V[r * nl * k:(r + 1) * nl * k],
        "W_sub": cat(Wsub) if Wsub else W[0:0],
        "R_sub": cat(Rsub) if Rsub else R[0:0],
        "B_sub": cat(Bsub) if Bsub else B[0:0],
        "W_root": W[((1 << q) - 2 + r) * t:((1 << q) - 1 + r) * t] if q >= 1 and pl >= 1 else W[0:0],
        "R_root": R[((1 << q) - 2 + r) * t:((1 << q) - 1 + r) * t] if q >= 1 and pl >= 1 else R[0:0],
        "W_top": W[0:((1 << q) - 2) * t] if q >= 2 else W[0:0],
        "R_top": R[0:((1 << q) - 2) * t] if q >= 2 else R[0:0],
        "B_top": B[0:((1 << q) - 1) * bb] if q >= 1 else B[0:0],
    }
    return out


def _cat_for(a):
    try:
        import torch
        if isinstance(a, torch.Tensor):
            return lambda xs: torch.cat(xs) if xs else a[0:0]
    except ImportError:  # pragma: no cover
        pass
    import numpy as np
    return lambda xs: np.concatenate(xs) if xs else a[0:0]


# ------------------------------------------------------------ communicator --

def unique_id() -> bytes:
    """A fresh NCCL unique id (HM_COMM_ID_BYTES bytes) from libhm (rank 0 calls this)."""
    buf = ctypes.create_string_buffer(HM_COMM_ID_BYTES)
    _check(_lib().hm_comm_unique_id(buf))
    return buf.raw


def broadcast_unique_id(group=None) -> bytes:
    """Rank 0's unique id on every rank of the torch.distributed group (the out-of-band
    step hm_comm_init leaves to the caller)."""
    import torch
    import torch.distributed as dist
    backend = dist.get_backend(group)
    device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.zeros(HM_COMM_ID_BYTES, dtype=torch.uint8, device=device)
    if dist.get_rank(group) == 0:
        t.copy_(torch.frombuffer(bytearray(unique_id()), dtype=torch.uint8))
    dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return bytes(t.cpu().tolist())


class Comm:
    """libhm's communicator (hm_comm*) for this process's current CUDA device."""

    def __init__(self, nranks: int, rank: int, uid: bytes):
        if len(uid) != HM_COMM_ID_BYTES:
            raise ValueError("unique id must have HM_COMM_ID_BYTES bytes")
        self.nranks, self.rank = int(nranks), int(rank)
        self._h = ctypes.c_void_p(None)
        _check(_lib().hm_comm_init(self.nranks, self.rank, uid, ctypes.byref(self._h)))

    @classmethod
    def from_group(cls, group=None) -> "Comm":
        import torch.distributed as dist
        return cls(dist.get_world_size(group), dist.get_rank(group), broadcast_unique_id(group))

    @property
    def handle(self):
        if not self._h:
            raise HmError(HM_ERR_INVALID_ARG, "communicator closed")
        return self._h

    def allgather(self, send, recv=None, stream=None):
        """recv[P * len(send)] <- every rank's send, rank order (hm_comm_allgather)."""
        import torch
        send = _dev(send, "send")
        with _on(stream):
            if recv is None:
                recv = torch.empty(self.nranks * send.numel(), dtype=torch.float64, device=send.device)
            _check(_lib().hm_comm_allgather(self.handle, _ptr(send), send.numel(), _ptr(recv), _stream(stream)))
        return recv

    def close(self):
        if self._h:
            h, self._h = self._h, ctypes.c_void_p(None)
            _check(_lib().hm_comm_destroy(h))

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


# ---------------------------------------------------------- one-call products --

def hodlr_dist_workspace_bytes(n, levels, leaf, ranks, nrhs, P) -> int:
    out = ctypes.c_size_t(0)
    t = make_tree(n, levels, leaf)
    _check(_lib().hm_hodlr_dist_workspace_bytes(ctypes.byref(t), _ranks(ranks, levels), int(nrhs), int(P),
                                                ctypes.byref(out)))
    return out.value


def hss_dist_workspace_bytes(n, levels, leaf, k, nrhs, P) -> int:
    out = ctypes.c_size_t(0)
    t = make_tree(n, levels, leaf)
    _check(_lib().hm_hss_dist_workspace_bytes(ctypes.byref(t), int(k), int(nrhs), int(P), ctypes.byref(out)))
    return out.value


def _local_xy(X_l, Y_l, n, P):
    import torch
    X_l = _dev(X_l, "X_local")
    if X_l.shape[0] != n // P:
        raise ValueError(f"X_local must have n/P = {n // P} rows, got {X_l.shape[0]}")
    if Y_l is None:
        Y_l = torch.empty_like(X_l)
    _dev(Y_l, "Y_local")
    if tuple(Y_l.shape) != tuple(X_l.shape):
        raise ValueError("Y_local shape != X_local shape")
    return X_l, Y_l, (1 if X_l.dim() == 1 else X_l.shape[1])


def hodlr_matvec_dist(comm: Comm, n, levels, leaf, ranks, D_l, U_l, V_l, X_l, Y_l=None, ws=None, stream=None):
    """Y_l = rows I_r of A X on this rank's GPU, one libhm call (hodlr_matvec_dist)."""
    import torch
    with _on(stream):
        X_l, Y_l, nrhs = _local_xy(X_l, Y_l, n, comm.nranks)
        for t_, nm in ((D_l, "D_local"), (U_l, "U_local"), (V_l, "V_local")):
            _dev(t_, nm)
        wsb = hodlr_dist_workspace_bytes(n, levels, leaf, ranks, nrhs, comm.nranks)
        if ws is None or ws.numel() < wsb:
            ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=X_l.device)
        t = make_tree(n, levels, leaf)
        _check(_lib().hodlr_matvec_dist(comm.handle, ctypes.byref(t), _ranks(ranks, levels), _ptr(D_l), _ptr(U_l),
                                        _ptr(V_l), _ptr(X_l), nrhs, _ptr(Y_l), ws.data_ptr(), ws.numel(),
                                        _stream(stream)))
    return Y_l


def hss_matvec_dist(comm: Comm, n, levels, leaf, k, sh, X_l, Y_l=None, ws=None, stream=None):
    """Y_l = rows I_r of A X for the HSS shard `sh` (hss_shard), one libhm call (hss_matvec_dist)."""
    import torch
    with _on(stream):
        X_l, Y_l, nrhs = _local_xy(X_l, Y_l, n, comm.nranks)
        for kk, v in sh.items():
            _dev(v, kk)
        wsb = hss_dist_workspace_bytes(n, levels, leaf, k, nrhs, comm.nranks)
        if ws is None or ws.numel() < wsb:
            ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=X_l.device)
        t = make_tree(n, levels, leaf)
        g = [_ptr(sh[a]) for a in ("D", "U", "V", "R_sub", "W_sub", "B_sub", "R_root", "W_root", "R_top", "W_top",
                                   "B_top")]
        _check(_lib().hss_matvec_dist(comm.handle, ctypes.byref(t), int(k), *g, _ptr(X_l), nrhs, _ptr(Y_l),
                                      ws.data_ptr(), ws.numel(), _stream(stream)))
    return Y_l


# ------------------------------------------------------- split-phase calls --

def hodlr_dist_sizes(n, levels, leaf, ranks, nrhs, P, r):
    lib = _lib()
    ws, sd = ctypes.c_size_t(0), ctypes.c_int64(0)
    t, part = make_tree(n, levels, leaf), hm_part(P, r)
    _check(lib.hm_hodlr_dist_sizes(ctypes.byref(t), _ranks(ranks, levels), int(nrhs), ctypes.byref(part),
                                   ctypes.byref(ws), ctypes.byref(sd)))
    return ws.value, sd.value


def hss_dist_sizes(n, levels, leaf, k, nrhs, P, r):
    lib = _lib()
    ws, sd = ctypes.c_size_t(0), ctypes.c_int64(0)
    t, part = make_tree(n, levels, leaf), hm_part(P, r)
    _check(lib.hm_hss_dist_sizes(ctypes.byref(t), int(k), int(nrhs), ctypes.byref(part), ctypes.byref(ws),
                                 ctypes.byref(sd)))
    return ws.value, sd.value


def hodlr_matvec_dist_begin(n, levels, leaf, ranks, P, r, V_l, X_l, send, ws, stream=None):
    t, part = make_tree(n, levels, leaf), hm_part(P, r)
    nrhs = 1 if X_l.dim() == 1 else X_l.shape[1]
    _check(_lib().hodlr_matvec_dist_begin(ctypes.byref(t), _ranks(ranks, levels), ctypes.byref(part), _ptr(V_l),
                                          _ptr(X_l), nrhs, _ptr(send), ws.data_ptr(), ws.numel(), _stream(stream)))


def hodlr_matvec_dist_local(n, levels, leaf, ranks, P, r, D_l, U_l, V_l, X_l, Y_l, ws, stream=None):
    t, part = make_tree(n, levels, leaf), hm_part(P, r)
    nrhs = 1 if X_l.dim() == 1 else X_l.shape[1]
    _check(_lib().hodlr_matvec_dist_local(ctypes.byref(t), _ranks(ranks, levels), ctypes.byref(part), _ptr(D_l),
                                          _ptr(U_l), _ptr(V_l), _ptr(X_l), nrhs, _ptr(Y_l), ws.data_ptr(),
                                          ws.numel(), _stream(stream)))


def hodlr_matvec_dist_end(n, levels, leaf, ranks, P, r, D_l, U_l, X_l, gathered, Y_l, ws, stream=None):
    t, part = make_tree(n, levels, leaf), hm_part(P, r)
    nrhs = 1 if X_l.dim() == 1 else X_l.shape[1]
    _check(_lib().hodlr_matvec_dist_end(ctypes.byref(t), _ranks(ranks, levels), ctypes.byref(part), _ptr(D_l),
                                        _ptr(U_l), _ptr(X_l), nrhs, _ptr(gathered), _ptr(Y_l), ws.data_ptr(),
                                        ws.numel(), _stream(stream)))


def hss_matvec_dist_begin(n, levels, leaf, k, P, r, sh, X_l, send, ws, stream=None):
    t, part = make_tree(n, levels, leaf), hm_part(P, r)
    nrhs = 1 if X_l.dim() == 1 else X_l.shape[1]
    _check(_lib().hss_matvec_dist_begin(ctypes.byref(t), int(k), ctypes.byref(part), _ptr(sh["V"]),
                                        _ptr(sh["W_sub"]), _ptr(sh["W_root"]), _ptr(X_l), nrhs, _ptr(send),
                                        ws.data_ptr(), ws.numel(), _stream(stream)))


def hss_matvec_dist_end(n, levels, leaf, k, P, r, sh, X_l, gathered, Y_l, ws, stream=None):
    t, part = make_tree(n, levels, leaf), hm_part(P, r)
    nrhs = 1 if X_l.dim() == 1 else X_l.shape[1]
    _check(_lib().hss_matvec_dist_end(ctypes.byref(t), int(k), ctypes.byref(part), _ptr(sh["D"]), _ptr(sh["U"]),
                                      _ptr(sh["R_sub"]), _ptr(sh["B_sub"]), _ptr(sh["R_root"]), _ptr(sh["W_top"]),
                                      _ptr(sh["R_top"]), _ptr(sh["B_top"]), _ptr(X_l), nrhs, _ptr(gathered),
                                      _ptr(Y_l), ws.data_ptr(), ws.numel(), _stream(stream)))
