"""B200-native HODLR / HSS matrix-(multi)vector product (hm-toolbox, arXiv 1909.07909).

Thin Python binding over the C-ABI library ``libhm.so`` (include/hm.h). It only
marshals arguments — torch tensors to device pointers, the tree to an
``hm_tree`` struct, torch's current CUDA stream to a ``cudaStream_t`` — and
allocates the workspace with torch. Every step of the product runs in the
library's sm_100a kernels. There is no CPU fallback: a missing library or a
non-CUDA tensor raises.

Names follow the C-ABI: ``hodlr_matvec``, ``hss_matvec`` (device tensors),
``hodlr_matvec_hostio``, ``hss_matvec_hostio`` (host X / Y, end-to-end path),
``hm_hodlr_workspace_bytes``, ``hm_hss_workspace_bytes``, ``hm_last_error``.
"""
from __future__ import annotations

import ctypes
import functools
import os
from typing import Optional, Sequence

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HM_LIBHM") or os.path.join(_PKG, "libhm.so")  # HM_LIBHM: dev variants only

HM_OK, HM_ERR_INVALID_ARG, HM_ERR_UNSUPPORTED, HM_ERR_WORKSPACE, HM_ERR_CUDA, HM_ERR_NCCL = 0, -1, -2, -3, -4, -5
HM_WS_HOSTIO = 1
_STATUS = {0: "HM_OK", -1: "HM_ERR_INVALID_ARG", -2: "HM_ERR_UNSUPPORTED", -3: "HM_ERR_WORKSPACE",
           -4: "HM_ERR_CUDA", -5: "HM_ERR_NCCL"}

# every symbol include/hm.h declares (tests check the library exports all of them)
EXPORTS = ("hm_hodlr_workspace_bytes", "hodlr_matvec", "hodlr_matvec_hostio", "hm_hss_workspace_bytes",
           "hss_matvec", "hss_matvec_hostio", "hm_last_error", "hm_abi_version", "hm_last_launch_count",
           "hm_profile_enable", "hm_profile_collect",
           "hm_hodlr_dist_sizes", "hodlr_matvec_dist_begin", "hodlr_matvec_dist_local", "hodlr_matvec_dist_end",
           "hm_hss_dist_sizes", "hss_matvec_dist_begin", "hss_matvec_dist_end",
           "hodlr_matvec_t", "hss_matvec_t",
           "hm_hodlr_norm2_workspace_bytes", "hodlr_norm2_est", "hm_hss_norm2_workspace_bytes", "hss_norm2_est",
           "hss_to_hodlr", "hm_hodlr_general_workspace_bytes", "hodlr_matvec_general",
           "hm_hss_general_workspace_bytes", "hss_matvec_general",
           "hm_comm_unique_id", "hm_comm_init", "hm_comm_destroy", "hm_comm_size", "hm_comm_allgather",
           "hm_hodlr_dist_workspace_bytes", "hodlr_matvec_dist", "hm_hss_dist_workspace_bytes", "hss_matvec_dist",
           "hm_hss_ranked_workspace_bytes", "hss_matvec_ranked",
           "hm_hss_noderanked_workspace_bytes", "hss_matvec_noderanked")


class HmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class hm_tree(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("levels", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("leaf", ctypes.c_int64)]


class hm_launch_record(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 40), ("call", ctypes.c_int32), ("ms", ctypes.c_float),
                ("start_ms", ctypes.c_float)]


_lib: Optional[ctypes.CDLL] = None


def load() -> ctypes.CDLL:
    """Load libhm.so (raises if it has not been built — there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if LIB_PATH == os.path.join(_PKG, "libhm.so"):
        # the in-tree library must carry the hash of the sources on disk (a stale
        # binary that travelled with a snapshot is rebuilt, never loaded)
        from . import build as _build
        if _build.needs_build():
            _build.build()
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not found: build it with `python -m paper_1909_07909_b200.build` "
                          "(the CUDA path has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    T = ctypes.POINTER(hm_tree)
    sigs = {
        "hm_hodlr_workspace_bytes": [T, P, i32, i32, ctypes.POINTER(sz)],
        "hodlr_matvec": [T, P, P, P, P, P, i32, P, P, sz, P],
        "hodlr_matvec_hostio": [T, P, P, P, P, P, i32, P, P, sz, P],
        "hodlr_matvec_t": [T, P, P, P, P, P, i32, P, P, sz, P],
        "hss_matvec_t": [T, i32, P, P, P, P, P, P, P, i32, P, P, sz, P],
        "hm_hss_workspace_bytes": [T, i32, i32, i32, ctypes.POINTER(sz)],
        "hss_matvec": [T, i32, P, P, P, P, P, P, P, i32, P, P, sz, P],
        "hss_matvec_hostio": [T, i32, P, P, P, P, P, P, P, i32, P, P, sz, P],
        "hm_hodlr_norm2_workspace_bytes": [T, P, ctypes.POINTER(sz)],
        "hodlr_norm2_est": [T, P, P, P, P, P, i32, P, P, sz, P],
        "hm_hss_norm2_workspace_bytes": [T, i32, ctypes.POINTER(sz)],
        "hss_norm2_est": [T, i32, P, P, P, P, P, P, P, i32, P, P, sz, P],
        "hss_to_hodlr": [T, i32, P, P, P, P, P, P, P, P],
        "hm_hodlr_general_workspace_bytes": [i64, i32, P, P, i32, ctypes.POINTER(sz)],
        "hodlr_matvec_general": [i64, i32, P, P, i32, P, P, P, P, i32, P, P, sz, P],
        "hm_hss_general_workspace_bytes": [i64, i32, P, i32, i32, ctypes.POINTER(sz)],
        "hss_matvec_general": [i64, i32, P, i32, i32, P, P, P, P, P, P, P, i32, P, P, sz, P],
        "hm_hss_ranked_workspace_bytes": [T, P, i32, ctypes.POINTER(sz)],
        "hss_matvec_ranked": [T, P, i32, P, P, P, P, P, P, P, i32, P, P, sz, P],
        "hm_hss_noderanked_workspace_bytes": [T, P, i32, ctypes.POINTER(sz)],
        "hss_matvec_noderanked": [T, P, i32, P, P, P, P, P, P, P, i32, P, P, sz, P],
        "hm_profile_enable": [i32],
        "hm_profile_collect": [ctypes.POINTER(hm_launch_record), i32, ctypes.POINTER(i32)],
    }
    for name, args in sigs.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    lib.hm_last_error.argtypes = []
    lib.hm_last_error.restype = ctypes.c_char_p
    lib.hm_abi_version.restype = ctypes.c_int32
    lib.hm_last_launch_count.restype = ctypes.c_int32
    _lib = lib
    return lib


def hm_last_error() -> str:
    return load().hm_last_error().decode()


def last_launch_count() -> int:
    return int(load().hm_last_launch_count())


def hm_profile_enable(on: bool = True) -> None:
    """Bracket every kernel launch with CUDA events on its stream (include/hm.h)."""
    _check(load().hm_profile_enable(1 if on else 0))


def hm_profile_collect(cap: int = 1 << 16):
    """[(kernel name, call index, ms)] in launch order; clears the trace."""
    return [(nm, c, ms) for nm, c, _, ms in hm_profile_timeline(cap)]


def hm_profile_timeline(cap: int = 1 << 16):
    """[(kernel name, call index, start_ms, ms)] in launch order, start_ms on one
    device timeline across streams (include/hm.h); clears the trace."""
    buf = (hm_launch_record * cap)()
    cnt = ctypes.c_int32(0)
    _check(load().hm_profile_collect(buf, cap, ctypes.byref(cnt)))
    return [(buf[i].name.decode(), int(buf[i].call), float(buf[i].start_ms), float(buf[i].ms))
            for i in range(min(cnt.value, cap))]


def _check(rc: int) -> None:
    if rc != HM_OK:
        raise HmError(rc, hm_last_error())


def make_tree(n: int, levels: int, leaf: int) -> hm_tree:
    return hm_tree(int(n), int(levels), 0, int(leaf))


def _ranks(ranks: Sequence[int], levels: int):
    """ranks[l-1] = k_l for l = 1..levels: exactly `levels` entries (a short list would
    silently turn the missing levels into zero blocks)."""
    ranks = [int(r) for r in ranks]
    if levels >= 0 and len(ranks) != levels:  # (negative depths are the library's to reject)
        raise ValueError(f"ranks has {len(ranks)} entries, need one per level ({levels})")
    return (ctypes.c_int32 * max(levels, 1, len(ranks)))(*(ranks or [0]))


def _numel_at_least(t, count, name):
    if t is not None and t.numel() < count:
        raise ValueError(f"{name} has {t.numel()} elements, the tree needs {count}")


def _xy(X, Y, n):
    """X [n] or [n][nrhs]; Y the same shape as X."""
    if X.shape[0] != n or X.dim() > 2:
        raise ValueError(f"X must be [n] or [n][nrhs] with n = {n}, got {tuple(X.shape)}")
    if Y is not None and tuple(Y.shape) != tuple(X.shape):
        raise ValueError(f"Y shape {tuple(Y.shape)} != X shape {tuple(X.shape)}")


def _hodlr_sizes(n, leaf, ranks, D, U, V):
    _numel_at_least(D, n * leaf, "D")
    kt = sum(int(r) for r in ranks)
    _numel_at_least(U, n * kt, "U")
    _numel_at_least(V, n * kt, "V")


def _hss_sizes(n, levels, leaf, k, D, U, V, R, W, B):
    _numel_at_least(D, n * leaf, "D")
    if k > 0 and levels > 0:
        _numel_at_least(U, n * k, "U")
        _numel_at_least(V, n * k, "V")
        _numel_at_least(B, ((1 << levels) - 1) * 2 * k * k, "B")
        if levels >= 2:
            _numel_at_least(R, ((1 << levels) - 2) * 2 * k * k, "R")
            _numel_at_least(W, ((1 << levels) - 2) * 2 * k * k, "W")


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    return t.data_ptr() if t.numel() > 0 else None


def _dev(t, name):
    import torch
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise TypeError(f"{name} must be a contiguous float64 CUDA tensor (no CPU fallback)")
    return t


def _stream(stream) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def hm_hodlr_workspace_bytes(n, levels, leaf, ranks, nrhs, flags=0) -> int:
    out = ctypes.c_size_t(0)
    t = make_tree(n, levels, leaf)
    _check(load().hm_hodlr_workspace_bytes(ctypes.byref(t), _ranks(ranks, levels), int(nrhs), int(flags),
                                           ctypes.byref(out)))
    return out.value


def hm_hss_workspace_bytes(n, levels, leaf, k, nrhs, flags=0) -> int:
    out = ctypes.c_size_t(0)
    t = make_tree(n, levels, leaf)
    _check(load().hm_hss_workspace_bytes(ctypes.byref(t), int(k), int(nrhs), int(flags), ctypes.byref(out)))
    return out.value


def _workspace(nbytes, workspace, device):
    import torch
    if workspace is None:
        workspace = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
    if workspace.numel() < nbytes:
        raise HmError(HM_ERR_WORKSPACE, f"workspace {workspace.numel()} < {nbytes} bytes")
    return workspace


def hodlr_matvec(n, levels, leaf, ranks, D, U, V, X, Y=None, workspace=None, stream=None, _fn="hodlr_matvec"):
    """Y = A X on the current CUDA stream for the HODLR matrix (D, U, V) (include/hm.h).
    X: [n][nrhs] (or [n]) float64 CUDA tensor. Returns Y (allocated if None)."""
    import torch
    X = _dev(X, "X")
    nrhs = 1 if X.dim() == 1 else X.shape[1]
    if Y is None:
        Y = torch.empty_like(X)
    _dev(Y, "Y"); _dev(D, "D"); _dev(U, "U"); _dev(V, "V")
    ws = _workspace(hm_hodlr_workspace_bytes(n, levels, leaf, ranks, nrhs), workspace, X.device)
    _xy(X, Y, n)
    _hodlr_sizes(n, leaf, ranks, D, U, V)
    t = make_tree(n, levels, leaf)
    _check(getattr(load(), _fn)(ctypes.byref(t), _ranks(ranks, levels), _ptr(D), _ptr(U), _ptr(V), _ptr(X), nrhs,
                                _ptr(Y), ws.data_ptr(), ws.numel(), _stream(stream)))
    return Y


def hodlr_matvec_t(n, levels, leaf, ranks, D, U, V, X, Y=None, workspace=None, stream=None):
    """Y = A^T X (adjoint, include/hm.h hodlr_matvec_t); arguments as hodlr_matvec."""
    return hodlr_matvec(n, levels, leaf, ranks, D, U, V, X, Y, workspace, stream, _fn="hodlr_matvec_t")


def hodlr_matvec_hostio(n, levels, leaf, ranks, D, U, V, X_host, Y_host, workspace=None, stream=None):
    """End-to-end variant: X_host / Y_host are (pinned) CPU float64 tensors; the library copies
    X in and Y out on the stream. The caller synchronises before reading Y_host."""
    import torch
    nrhs = 1 if X_host.dim() == 1 else X_host.shape[1]
    for t_, nm in ((X_host, "X_host"), (Y_host, "Y_host")):
        if t_.is_cuda or t_.dtype != torch.float64 or not t_.is_contiguous():
            raise TypeError(f"{nm} must be a contiguous float64 host tensor")
    _dev(D, "D"); _dev(U, "U"); _dev(V, "V")
    ws = _workspace(hm_hodlr_workspace_bytes(n, levels, leaf, ranks, nrhs, HM_WS_HOSTIO), workspace, D.device)
    _xy(X_host, Y_host, n)
    _hodlr_sizes(n, leaf, ranks, D, U, V)
    t = make_tree(n, levels, leaf)
    _check(load().hodlr_matvec_hostio(ctypes.byref(t), _ranks(ranks, levels), _ptr(D), _ptr(U), _ptr(V),
                                      X_host.data_ptr(), nrhs, Y_host.data_ptr(), ws.data_ptr(), ws.numel(),
                                      _stream(stream)))
    return Y_host


def hss_matvec_t(n, levels, leaf, k, D, U, V, R, W, B, X, Y=None, workspace=None, stream=None):
    """Y = A^T X (adjoint, include/hm.h hss_matvec_t); arguments as hss_matvec."""
    return hss_matvec(n, levels, leaf, k, D, U, V, R, W, B, X, Y, workspace, stream, _fn="hss_matvec_t")


def hss_matvec(n, levels, leaf, k, D, U, V, R, W, B, X, Y=None, workspace=None, stream=None, _fn="hss_matvec"):
    """Y = A X on the current CUDA stream for the HSS matrix (D, U, V, R, W, B) (include/hm.h)."""
    import torch
    X = _dev(X, "X")
    nrhs = 1 if X.dim() == 1 else X.shape[1]
    if Y is None:
        Y = torch.empty_like(X)
    for t_, nm in ((Y, "Y"), (D, "D"), (U, "U"), (V, "V"), (R, "R"), (W, "W"), (B, "B")):
        _dev(t_, nm)
    ws = _workspace(hm_hss_workspace_bytes(n, levels, leaf, k, nrhs), workspace, X.device)
    _xy(X, Y, n)
    _hss_sizes(n, levels, leaf, k, D, U, V, R, W, B)
    t = make_tree(n, levels, leaf)
    _check(getattr(load(), _fn)(ctypes.byref(t), int(k), _ptr(D), _ptr(U), _ptr(V), _ptr(R), _ptr(W), _ptr(B),
                                _ptr(X), nrhs, _ptr(Y), ws.data_ptr(), ws.numel(), _stream(stream)))
    return Y


def hss_matvec_hostio(n, levels, leaf, k, D, U, V, R, W, B, X_host, Y_host, workspace=None, stream=None):
    import torch
    nrhs = 1 if X_host.dim() == 1 else X_host.shape[1]
    for t_, nm in ((X_host, "X_host"), (Y_host, "Y_host")):
        if t_.is_cuda or t_.dtype != torch.float64 or not t_.is_contiguous():
            raise TypeError(f"{nm} must be a contiguous float64 host tensor")
    for t_, nm in ((D, "D"), (U, "U"), (V, "V"), (R, "R"), (W, "W"), (B, "B")):
        _dev(t_, nm)
    ws = _workspace(hm_hss_workspace_bytes(n, levels, leaf, k, nrhs, HM_WS_HOSTIO), workspace, D.device)
    _xy(X_host, Y_host, n)
    _hss_sizes(n, levels, leaf, k, D, U, V, R, W, B)
    t = make_tree(n, levels, leaf)
    _check(load().hss_matvec_hostio(ctypes.byref(t), int(k), _ptr(D), _ptr(U), _ptr(V), _ptr(R), _ptr(W), _ptr(B),
                                    X_host.data_ptr(), nrhs, Y_host.data_ptr(), ws.data_ptr(), ws.numel(),
                                    _stream(stream)))
    return Y_host


# ------------------------------------------------- ||A||_2 estimate (f2) --

def hm_hodlr_norm2_workspace_bytes(n, levels, leaf, ranks) -> int:
    out = ctypes.c_size_t(0)
    t = make_tree(n, levels, leaf)
    _check(load().hm_hodlr_norm2_workspace_bytes(ctypes.byref(t), _ranks(ranks, levels), ctypes.byref(out)))
    return out.value


def hm_hss_norm2_workspace_bytes(n, levels, leaf, k) -> int:
    out = ctypes.c_size_t(0)
    t = make_tree(n, levels, leaf)
    _check(load().hm_hss_norm2_workspace_bytes(ctypes.byref(t), int(k), ctypes.byref(out)))
    return out.value


def _est(est, device):
    import torch
    if est is None:
        est = torch.zeros(1, dtype=torch.float64, device=device)
    return _dev(est, "est")


def hodlr_norm2_est(n, levels, leaf, ranks, D, U, V, x0, iters, est=None, workspace=None, stream=None):
    """||A||_2 estimate (power method on A A^*, include/hm.h hodlr_norm2_est): returns a 1-element
    float64 CUDA tensor written asynchronously on the stream."""
    x0 = _dev(x0, "x0")
    _dev(D, "D"); _dev(U, "U"); _dev(V, "V")
    est = _est(est, x0.device)
    ws = _workspace(hm_hodlr_norm2_workspace_bytes(n, levels, leaf, ranks), workspace, x0.device)
    _numel_at_least(x0, n, "x0")
    _hodlr_sizes(n, leaf, ranks, D, U, V)
    t = make_tree(n, levels, leaf)
    _check(load().hodlr_norm2_est(ctypes.byref(t), _ranks(ranks, levels), _ptr(D), _ptr(U), _ptr(V), _ptr(x0),
                                  int(iters), _ptr(est), ws.data_ptr(), ws.numel(), _stream(stream)))
    return est


def hss_norm2_est(n, levels, leaf, k, D, U, V, R, W, B, x0, iters, est=None, workspace=None, stream=None):
    """||A||_2 estimate of an HSS matrix (include/hm.h hss_norm2_est)."""
    x0 = _dev(x0, "x0")
    for t_, nm in ((D, "D"), (U, "U"), (V, "V"), (R, "R"), (W, "W"), (B, "B")):
        _dev(t_, nm)
    est = _est(est, x0.device)
    ws = _workspace(hm_hss_norm2_workspace_bytes(n, levels, leaf, k), workspace, x0.device)
    _numel_at_least(x0, n, "x0")
    _hss_sizes(n, levels, leaf, k, D, U, V, R, W, B)
    t = make_tree(n, levels, leaf)
    _check(load().hss_norm2_est(ctypes.byref(t), int(k), _ptr(D), _ptr(U), _ptr(V), _ptr(R), _ptr(W), _ptr(B),
                                _ptr(x0), int(iters), _ptr(est), ws.data_ptr(), ws.numel(), _stream(stream)))
    return est


# ---------------------------------------------------------- hss2hodlr (f3) --

def hss_to_hodlr(n, levels, leaf, k, U, V, R, W, B, Uh=None, Vh=None, stream=None):
    """Exact HODLR factors (Uh, Vh), level-major [levels][n][k], of an HSS matrix (include/hm.h
    hss_to_hodlr). The HODLR leaf blocks are the HSS D; ranks are [k] * levels."""
    import torch
    U = _dev(U, "U")
    for t_, nm in ((V, "V"), (R, "R"), (W, "W"), (B, "B")):
        _dev(t_, nm)
    _hss_sizes(n, levels, leaf, k, None, U, V, R, W, B)
    size = max(levels, 0) * n * k
    if Uh is None:
        Uh = torch.empty(size, dtype=torch.float64, device=U.device)
    if Vh is None:
        Vh = torch.empty(size, dtype=torch.float64, device=U.device)
    _dev(Uh, "Uh"); _dev(Vh, "Vh")
    _numel_at_least(Uh, size, "Uh")
    _numel_at_least(Vh, size, "Vh")
    t = make_tree(n, levels, leaf)
    _check(load().hss_to_hodlr(ctypes.byref(t), int(k), _ptr(U), _ptr(V), _ptr(R), _ptr(W), _ptr(B), _ptr(Uh),
                               _ptr(Vh), _stream(stream)))
    return Uh, Vh


# ------------------------------------------------------ general trees (f4) --

def _endpoints(c, levels):
    import numpy as np
    c = np.ascontiguousarray(c, dtype=np.int64)
    if c.shape != (1 << levels,):
        raise ValueError("endpoint vector must have 2^levels entries")
    return c


def _leaf_block_doubles(c) -> int:
    """sum_i |I_i|^2 (the leaf blocks D_i) for the endpoint vector c."""
    import numpy as np
    sizes = np.diff(np.asarray(c, dtype=np.int64), prepend=np.int64(0))
    return int(np.dot(sizes, sizes))


def hm_hodlr_general_workspace_bytes(n, levels, c, ranks, nrhs) -> int:
    c = _endpoints(c, levels)
    out = ctypes.c_size_t(0)
    _check(load().hm_hodlr_general_workspace_bytes(int(n), int(levels), c.ctypes.data, _ranks(ranks, levels),
                                                   int(nrhs), ctypes.byref(out)))
    return out.value


def hodlr_matvec_general(n, levels, c, ranks, D, U, V, X, op=0, Y=None, workspace=None, stream=None):
    """Y = A X (op 0) or A^T X (op 1) for a HODLR matrix on the tree with leaf endpoints c (host,
    2^levels int64), per-level ranks allowed (include/hm.h hodlr_matvec_general)."""
    import torch
    c = _endpoints(c, levels)
    X = _dev(X, "X")
    nrhs = 1 if X.dim() == 1 else X.shape[1]
    if Y is None:
        Y = torch.empty_like(X)
    _dev(Y, "Y"); _dev(D, "D"); _dev(U, "U"); _dev(V, "V")
    ws = _workspace(hm_hodlr_general_workspace_bytes(n, levels, c, ranks, nrhs), workspace, X.device)
    _xy(X, Y, n)
    _numel_at_least(D, _leaf_block_doubles(c), "D")
    kt = sum(int(r) for r in ranks)
    _numel_at_least(U, n * kt, "U")
    _numel_at_least(V, n * kt, "V")
    _check(load().hodlr_matvec_general(int(n), int(levels), c.ctypes.data, _ranks(ranks, levels), int(op), _ptr(D),
                                       _ptr(U), _ptr(V), _ptr(X), nrhs, _ptr(Y), ws.data_ptr(), ws.numel(),
                                       _stream(stream)))
    return Y


def hm_hss_general_workspace_bytes(n, levels, c, k, nrhs) -> int:
    c = _endpoints(c, levels)
    out = ctypes.c_size_t(0)
    _check(load().hm_hss_general_workspace_bytes(int(n), int(levels), c.ctypes.data, int(k), int(nrhs),
                                                 ctypes.byref(out)))
    return out.value


def hss_matvec_general(n, levels, c, k, D, U, V, R, W, B, X, op=0, Y=None, workspace=None, stream=None):
    """Y = A X (op 0) or A^T X (op 1) for an HSS matrix on the tree with leaf endpoints c."""
    import torch
    c = _endpoints(c, levels)
    X = _dev(X, "X")
    nrhs = 1 if X.dim() == 1 else X.shape[1]
    if Y is None:
        Y = torch.empty_like(X)
    for t_, nm in ((Y, "Y"), (D, "D"), (U, "U"), (V, "V"), (R, "R"), (W, "W"), (B, "B")):
        _dev(t_, nm)
    ws = _workspace(hm_hss_general_workspace_bytes(n, levels, c, k, nrhs), workspace, X.device)
    _xy(X, Y, n)
    _hss_sizes(n, levels, 0, k, None, U, V, R, W, B)
    _numel_at_least(D, _leaf_block_doubles(c), "D")
    _check(load().hss_matvec_general(int(n), int(levels), c.ctypes.data, int(k), int(op), _ptr(D), _ptr(U), _ptr(V),
                                     _ptr(R), _ptr(W), _ptr(B), _ptr(X), nrhs, _ptr(Y), ws.data_ptr(), ws.numel(),
                                     _stream(stream)))
    return Y


# ------------------------------------------------ HSS, per-level ranks (f4) --

def hss_ranked_sizes(n, levels, ranks):
    """Generator sizes (doubles) of an HSS matrix with per-level ranks (include/hm.h
    hss_matvec_ranked): U/V, R/W, B."""
    k = [int(r) for r in ranks]
    kp = k[-1] if levels else 0
    rw = sum((1 << l) * 2 * k[l] * k[l - 1] for l in range(1, levels))
    b = sum((1 << (l - 1)) * 2 * k[l - 1] ** 2 for l in range(1, levels + 1))
    return n * kp, rw, b


def hm_hss_ranked_workspace_bytes(n, levels, leaf, ranks, nrhs) -> int:
    out = ctypes.c_size_t(0)
    t = make_tree(n, levels, leaf)
    _check(load().hm_hss_ranked_workspace_bytes(ctypes.byref(t), _ranks(ranks, levels), int(nrhs),
                                                ctypes.byref(out)))
    return out.value


def hss_matvec_ranked(n, levels, leaf, ranks, D, U, V, R, W, B, X, op=0, Y=None, workspace=None, stream=None):
    """Y = A X (op 0) or A^T X (op 1) for an HSS matrix with per-level ranks k_l = ranks[l-1]
    (include/hm.h hss_matvec_ranked)."""
    import torch
    X = _dev(X, "X")
    nrhs = 1 if X.dim() == 1 else X.shape[1]
    if Y is None:
        Y = torch.empty_like(X)
    for t_, nm in ((Y, "Y"), (D, "D"), (U, "U"), (V, "V"), (R, "R"), (W, "W"), (B, "B")):
        _dev(t_, nm)
    ws = _workspace(hm_hss_ranked_workspace_bytes(n, levels, leaf, ranks, nrhs), workspace, X.device)
    _xy(X, Y, n)
    nuv, nrw, nb = hss_ranked_sizes(n, levels, ranks)
    _numel_at_least(D, n * leaf, "D")
    for t_, c_, nm in ((U, nuv, "U"), (V, nuv, "V"), (R, nrw, "R"), (W, nrw, "W"), (B, nb, "B")):
        _numel_at_least(t_, c_, nm)
    t = make_tree(n, levels, leaf)
    _check(load().hss_matvec_ranked(ctypes.byref(t), _ranks(ranks, levels), int(op), _ptr(D), _ptr(U), _ptr(V),
                                    _ptr(R), _ptr(W), _ptr(B), _ptr(X), nrhs, _ptr(Y), ws.data_ptr(), ws.numel(),
                                    _stream(stream)))
    return Y


# ------------------------------------------------- HSS, per-node ranks (f4) --

def _kn_key(node_ranks) -> bytes:
    import numpy as np
    if isinstance(node_ranks, np.ndarray) and node_ranks.dtype == np.int32 and node_ranks.flags.c_contiguous:
        return node_ranks.tobytes()  # (a list of 2^(p+1) ranks costs ~1 ms to convert: pass an int32 array)
    return np.ascontiguousarray(node_ranks, dtype=np.int32).tobytes()


def hss_noderanked_sizes(n, levels, leaf, node_ranks):
    """Generator sizes (doubles) of an HSS matrix with per-node ranks (include/hm.h
    hss_matvec_noderanked): U/V, R/W, B."""
    return _noderanked_sizes(int(n), int(levels), int(leaf), _kn_key(node_ranks))


@functools.lru_cache(maxsize=16)
def _noderanked_sizes(n, levels, leaf, key):
    import numpy as np
    kn = np.frombuffer(key, dtype=np.int32).tolist()
    h = lambda l, i: (1 << l) - 2 + i  # noqa: E731
    nuv = sum(leaf * kn[h(levels, i)] for i in range(1 << levels)) if levels else 0
    nrw = sum((kn[h(l + 1, 2 * i)] + kn[h(l + 1, 2 * i + 1)]) * kn[h(l, i)]
              for l in range(1, levels) for i in range(1 << l))
    nb = sum(2 * kn[h(l, 2 * q)] * kn[h(l, 2 * q + 1)] for l in range(1, levels + 1) for q in range(1 << (l - 1)))
    return nuv, nrw, nb


def _node_ranks(node_ranks, levels):
    return _node_ranks_c(_kn_key(node_ranks), int(levels))


@functools.lru_cache(maxsize=16)
def _node_ranks_c(key, levels):
    import numpy as np
    nr = np.frombuffer(key, dtype=np.int32).tolist()
    need = (1 << (levels + 1)) - 2
    if len(nr) != need:
        raise ValueError(f"node_ranks has {len(nr)} entries, need 2^(levels+1) - 2 = {need}")
    return (ctypes.c_int32 * max(need, 1))(*(nr or [0]))


def hm_hss_noderanked_workspace_bytes(n, levels, leaf, node_ranks, nrhs) -> int:
    out = ctypes.c_size_t(0)
    t = make_tree(n, levels, leaf)
    _check(load().hm_hss_noderanked_workspace_bytes(ctypes.byref(t), _node_ranks(node_ranks, levels), int(nrhs),
                                                    ctypes.byref(out)))
    return out.value


def hss_matvec_noderanked(n, levels, leaf, node_ranks, D, U, V, R, W, B, X, op=0, Y=None, workspace=None,
                          stream=None):
    """Y = A X (op 0) or A^T X (op 1) for an HSS matrix with per-node ranks (
    include/hm.h hss_matvec_noderanked); node (l, i) at heap index 2^l - 2 + i."""
    import torch
    X = _dev(X, "X")
    nrhs = 1 if X.dim() == 1 else X.shape[1]
    if Y is None:
        Y = torch.empty_like(X)
    for t_, nm in ((Y, "Y"), (D, "D"), (U, "U"), (V, "V"), (R, "R"), (W, "W"), (B, "B")):
        _dev(t_, nm)
    ws = _workspace(hm_hss_noderanked_workspace_bytes(n, levels, leaf, node_ranks, nrhs), workspace, X.device)
    _xy(X, Y, n)
    nuv, nrw, nb = hss_noderanked_sizes(n, levels, leaf, node_ranks)
    _numel_at_least(D, n * leaf, "D")
    for t_, c_, nm in ((U, nuv, "U"), (V, nuv, "V"), (R, nrw, "R"), (W, nrw, "W"), (B, nb, "B")):
        _numel_at_least(t_, c_, nm)
    t = make_tree(n, levels, leaf)
    _check(load().hss_matvec_noderanked(ctypes.byref(t), _node_ranks(node_ranks, levels), int(op), _ptr(D), _ptr(U),
                                        _ptr(V), _ptr(R), _ptr(W), _ptr(B), _ptr(X), nrhs, _ptr(Y), ws.data_ptr(),
                                        ws.numel(), _stream(stream)))
    return Y
