"""Multi-GPU HODLR / HSS matvec: one process per GPU, P = 2^q ranks.

Rank r owns the rows of the level-q node (q, r) and its whole subtree; the only
exchange is one allgather (NCCL over NVLink through torch.distributed) of
  HODLR: the rank's partial top-level products V_l(I_r)^T X(I_r), l = 1..q;
  HSS:   the x block of node (q, r) (Step 1 up to the subtree root).
Every compute step runs in libhm (include/hm.h, the *_dist_* calls); this module
only shards the generators (index arithmetic), allocates buffers with torch and
issues the collective. The HODLR allgather is overlapped with the subtree's
V^T X pass (hodlr_matvec_dist_local).
"""
from __future__ import annotations

import ctypes
from typing import Sequence

from . import (_check, _dev, _ptr, _ranks, _stream, hm_tree, load, make_tree)


class hm_part(ctypes.Structure):
    _fields_ = [("nranks", ctypes.c_int32), ("rank", ctypes.c_int32)]


_sigs_done = False


def _lib():
    global _sigs_done
    lib = load()
    if not _sigs_done:
        P, i32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_size_t
        T, PT = ctypes.POINTER(hm_tree), ctypes.POINTER(hm_part)
        sigs = {
            "hm_hodlr_dist_sizes": [T, P, i32, PT, ctypes.POINTER(sz), ctypes.POINTER(ctypes.c_int64)],
            "hodlr_matvec_dist_begin": [T, P, PT, P, P, i32, P, P, sz, P],
            "hodlr_matvec_dist_local": [T, P, PT, P, P, i32, P, sz, P],
            "hodlr_matvec_dist_end": [T, P, PT, P, P, P, i32, P, P, P, sz, P],
            "hm_hss_dist_sizes": [T, i32, i32, PT, ctypes.POINTER(sz), ctypes.POINTER(ctypes.c_int64)],
            "hss_matvec_dist_begin": [T, i32, PT, P, P, P, P, i32, P, P, sz, P],
            "hss_matvec_dist_end": [T, i32, PT, P, P, P, P, P, P, P, P, P, i32, P, P, P, sz, P],
        }
        for name, args in sigs.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        _sigs_done = True
    return lib


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


# ---------------------------------------------------------------- the calls --

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


def hodlr_matvec_dist_local(n, levels, leaf, ranks, P, r, V_l, X_l, ws, stream=None):
    t, part = make_tree(n, levels, leaf), hm_part(P, r)
    nrhs = 1 if X_l.dim() == 1 else X_l.shape[1]
    _check(_lib().hodlr_matvec_dist_local(ctypes.byref(t), _ranks(ranks, levels), ctypes.byref(part), _ptr(V_l),
                                          _ptr(X_l), nrhs, ws.data_ptr(), ws.numel(), _stream(stream)))


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


def allgather(send, gathered, group=None, async_op=False):
    """gathered[P * len(send)] <- concat over ranks of send, rank order (NCCL on GPU,
    gloo on CPU)."""
    import torch.distributed as dist
    if send.numel() == 0:
        return None
    return dist.all_gather_into_tensor(gathered, send, group=group, async_op=async_op)


def hodlr_matvec_dist(n, levels, leaf, ranks, D_l, U_l, V_l, X_l, Y_l=None, group=None, ws=None, stream=None):
    """Y_l = rows I_r of A X, on this rank's GPU (one process per GPU)."""
    import torch
    import torch.distributed as dist
    P, r = dist.get_world_size(group), dist.get_rank(group)
    X_l = _dev(X_l, "X_local")
    nrhs = 1 if X_l.dim() == 1 else X_l.shape[1]
    if Y_l is None:
        Y_l = torch.empty_like(X_l)
    wsb, sd = hodlr_dist_sizes(n, levels, leaf, ranks, nrhs, P, r)
    if ws is None or ws.numel() < wsb:
        ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=X_l.device)
    send = torch.empty(max(sd, 1), dtype=torch.float64, device=X_l.device)[:sd]
    gathered = torch.empty(max(P * sd, 1), dtype=torch.float64, device=X_l.device)[:P * sd]
    hodlr_matvec_dist_begin(n, levels, leaf, ranks, P, r, V_l, X_l, send, ws, stream)
    work = allgather(send, gathered, group, async_op=True)  # overlaps the subtree V^T X pass
    hodlr_matvec_dist_local(n, levels, leaf, ranks, P, r, V_l, X_l, ws, stream)
    if work is not None:
        work.wait()
    hodlr_matvec_dist_end(n, levels, leaf, ranks, P, r, D_l, U_l, X_l, gathered, Y_l, ws, stream)
    return Y_l


def hss_matvec_dist(n, levels, leaf, k, sh, X_l, Y_l=None, group=None, ws=None, stream=None):
    """Y_l = rows I_r of A X for the HSS shard `sh` (hss_shard)."""
    import torch
    import torch.distributed as dist
    P, r = dist.get_world_size(group), dist.get_rank(group)
    X_l = _dev(X_l, "X_local")
    nrhs = 1 if X_l.dim() == 1 else X_l.shape[1]
    if Y_l is None:
        Y_l = torch.empty_like(X_l)
    wsb, sd = hss_dist_sizes(n, levels, leaf, k, nrhs, P, r)
    if ws is None or ws.numel() < wsb:
        ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=X_l.device)
    send = torch.empty(max(sd, 1), dtype=torch.float64, device=X_l.device)[:sd]
    gathered = torch.empty(max(P * sd, 1), dtype=torch.float64, device=X_l.device)[:P * sd]
    hss_matvec_dist_begin(n, levels, leaf, k, P, r, sh, X_l, send, ws, stream)
    allgather(send, gathered, group)
    hss_matvec_dist_end(n, levels, leaf, k, P, r, sh, X_l, gathered, Y_l, ws, stream)
    return Y_l
