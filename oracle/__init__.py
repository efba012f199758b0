"""CPU oracle for the HODLR / HSS matrix-(multi)vector product (hm-toolbox, arXiv 1909.07909).

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this package. The product path (``paper_1909_07909_b200``) never imports it,
and this package never imports the product: they share no code. Inputs for
both come from ``hm_inputs`` (seeded generators, no arithmetic of the method).

The arithmetic lives in ``hm_oracle.c`` (plain C, fp64, sequential sums in
natural order, ``-ffp-contract=off``); this module only marshals numpy arrays
into it with ctypes. See ``hm_oracle.h`` for layouts and the paper passages
(PAPER.md line numbers) each routine follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib: Optional[ctypes.CDLL] = None

_CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-Wall"]
_LDLIBS = ["-lm"]


def build(force: bool = False) -> str:
    """Compile hm_oracle.c into liboracle.so (gcc). Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "hm_oracle.h"))
    ):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *_CFLAGS, "-o", tmp, _SRC, *_LDLIBS])
        os.replace(tmp, _LIB)
    return _LIB


def _load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64, i32 = ctypes.c_int64, ctypes.c_int32
        sig = {
            "oracle_default_cluster": [i64, i64, P, P, i64],
            "oracle_hodlr_matvec": [i64, i32, P, P, P, P, P, P, i32, P],
            "oracle_hodlr_matvec_leaves": [i64, i32, P, P, P, P, P, P, i32, P, i64, P],
            "oracle_hss_matvec": [i64, i32, P, i32, P, P, P, P, P, P, P, i32, P],
            "oracle_hss_matvec_leaves": [i64, i32, P, i32, P, P, P, P, P, P, P, i32, P, i64, P],
            "oracle_hodlr_dense": [i64, i32, P, P, P, P, P, P],
            "oracle_hss_dense": [i64, i32, P, i32, P, P, P, P, P, P, P],
            "oracle_dense_matvec": [i64, P, P, i32, P],
            "oracle_laplacian_inverse_apply": [i64, P, i32, P],
            "oracle_num_threads": [],
            "oracle_hodlr_matvec_t": [i64, i32, P, P, P, P, P, P, i32, P],
            "oracle_hodlr_matvec_t_leaves": [i64, i32, P, P, P, P, P, P, i32, P, i64, P],
            "oracle_hss_matvec_t": [i64, i32, P, i32, P, P, P, P, P, P, P, i32, P],
            "oracle_hss_matvec_t_leaves": [i64, i32, P, i32, P, P, P, P, P, P, P, i32, P, i64, P],
            "oracle_hodlr_norm2_est": [i64, i32, P, P, P, P, P, P, i32, P],
            "oracle_hss_norm2_est": [i64, i32, P, i32, P, P, P, P, P, P, P, i32, P],
            "oracle_hss_to_hodlr": [i64, i32, P, i32, P, P, P, P, P, P, P],
            "oracle_hss_matvec_ranked": [i64, i32, P, P, P, P, P, P, P, P, P, i32, P],
            "oracle_hss_matvec_ranked_t": [i64, i32, P, P, P, P, P, P, P, P, P, i32, P],
            "oracle_hss_dense_ranked": [i64, i32, P, P, P, P, P, P, P, P, P],
            "oracle_hss_matvec_noderanked": [i64, i32, P, P, P, P, P, P, P, P, P, i32, P],
            "oracle_hss_matvec_noderanked_t": [i64, i32, P, P, P, P, P, P, P, P, P, i32, P],
            "oracle_hss_dense_noderanked": [i64, i32, P, P, P, P, P, P, P, P, P],
        }
        for name, args in sig.items():
            f = getattr(_lib, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        _lib.oracle_set_num_threads.argtypes = [ctypes.c_int]
        _lib.oracle_set_num_threads.restype = None
    return _lib


def _f64(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def _check(rc: int, name: str) -> None:
    if rc != 0:
        raise ValueError(f"{name}: invalid arguments (rc={rc})")


def _tree(n: int, p: int, c: Optional[Sequence[int]]) -> np.ndarray:
    if c is None:
        if n % (1 << p):
            raise ValueError("uniform tree needs n divisible by 2^p")
        b = n >> p
        c = [(i + 1) * b for i in range(1 << p)]
    c = np.ascontiguousarray(c, dtype=np.int64)
    if c.shape != (1 << p,):
        raise ValueError("endpoint vector must have 2^p entries")
    return c


def num_threads() -> int:
    return _load().oracle_num_threads()


def set_num_threads(n: int) -> None:
    """OpenMP threads of the oracle's loops (results are bitwise independent of it)."""
    _load().oracle_set_num_threads(int(n))


def default_cluster(n: int, nmin: int):
    """(p, c) of the default tree."""
    lib = _load()
    p = ctypes.c_int32(0)
    _check(lib.oracle_default_cluster(n, nmin, ctypes.addressof(p), None, 0), "default_cluster")
    c = np.zeros(1 << p.value, dtype=np.int64)
    _check(lib.oracle_default_cluster(n, nmin, ctypes.addressof(p), _ptr(c), c.size), "default_cluster")
    return p.value, c


def _X2(X):
    X = _f64(X)
    if X.ndim == 1:
        X = X[:, None]
    return X


def hodlr_matvec(n, p, ranks, D, U, V, X, c=None) -> np.ndarray:
    """Y = A X, Fig. 5 left."""
    c = _tree(n, p, c)
    X = _X2(X)
    m = X.shape[1]
    ranks = np.ascontiguousarray(ranks if p > 0 else [0], dtype=np.int32)
    D, U, V = _f64(D), _f64(U), _f64(V)
    Y = np.empty((n, m), dtype=np.float64)
    rc = _load().oracle_hodlr_matvec(n, p, _ptr(c), _ptr(ranks), _ptr(D), _ptr(U), _ptr(V), _ptr(X), m, _ptr(Y))
    _check(rc, "hodlr_matvec")
    return Y


def hodlr_matvec_leaves(n, p, ranks, Dsel, U, V, X, leaves, c=None) -> np.ndarray:
    """Rows of Y = A X for the listed leaves only (same arithmetic, same order)."""
    c = _tree(n, p, c)
    X = _X2(X)
    m = X.shape[1]
    ranks = np.ascontiguousarray(ranks if p > 0 else [0], dtype=np.int32)
    leaves = np.ascontiguousarray(leaves, dtype=np.int64)
    rows = sum(int(c[L] - (c[L - 1] if L > 0 else 0)) for L in leaves)
    Dsel, U, V = _f64(Dsel), _f64(U), _f64(V)
    Y = np.empty((rows, m), dtype=np.float64)
    rc = _load().oracle_hodlr_matvec_leaves(
        n, p, _ptr(c), _ptr(ranks), _ptr(Dsel), _ptr(U), _ptr(V), _ptr(X), m, _ptr(leaves), leaves.size, _ptr(Y)
    )
    _check(rc, "hodlr_matvec_leaves")
    return Y


def hss_matvec(n, p, k, D, U, V, R, W, B, X, c=None) -> np.ndarray:
    """Y = A X, Fig. 5 right, readings G1/G2."""
    c = _tree(n, p, c)
    X = _X2(X)
    m = X.shape[1]
    D, U, V, R, W, B = (_f64(a) for a in (D, U, V, R, W, B))
    Y = np.empty((n, m), dtype=np.float64)
    rc = _load().oracle_hss_matvec(
        n, p, _ptr(c), k, _ptr(D), _ptr(U), _ptr(V), _ptr(R), _ptr(W), _ptr(B), _ptr(X), m, _ptr(Y)
    )
    _check(rc, "hss_matvec")
    return Y


def hss_matvec_leaves(n, p, k, Dsel, U, V, R, W, B, X, leaves, c=None) -> np.ndarray:
    c = _tree(n, p, c)
    X = _X2(X)
    m = X.shape[1]
    leaves = np.ascontiguousarray(leaves, dtype=np.int64)
    rows = sum(int(c[L] - (c[L - 1] if L > 0 else 0)) for L in leaves)
    Dsel, U, V, R, W, B = (_f64(a) for a in (Dsel, U, V, R, W, B))
    Y = np.empty((rows, m), dtype=np.float64)
    rc = _load().oracle_hss_matvec_leaves(
        n, p, _ptr(c), k, _ptr(Dsel), _ptr(U), _ptr(V), _ptr(R), _ptr(W), _ptr(B), _ptr(X), m,
        _ptr(leaves), leaves.size, _ptr(Y)
    )
    _check(rc, "hss_matvec_leaves")
    return Y


def hss_matvec_ranked(n, p, ranks, D, U, V, R, W, B, X, c=None, trans=False) -> np.ndarray:
    """Y = A X (A^T X if trans) for an HSS matrix with per-level ranks k_l = ranks[l-1]
    (P:264), Fig. 5 right; layout in hm_oracle.h."""
    c = _tree(n, p, c)
    X = _X2(X)
    m = X.shape[1]
    ranks = np.ascontiguousarray(ranks if p > 0 else [0], dtype=np.int32)
    D, U, V, R, W, B = (_f64(a) for a in (D, U, V, R, W, B))
    Y = np.empty((n, m), dtype=np.float64)
    fn = _load().oracle_hss_matvec_ranked_t if trans else _load().oracle_hss_matvec_ranked
    rc = fn(n, p, _ptr(c), _ptr(ranks), _ptr(D), _ptr(U), _ptr(V), _ptr(R), _ptr(W), _ptr(B), _ptr(X), m, _ptr(Y))
    _check(rc, "hss_matvec_ranked")
    return Y


def hss_dense_ranked(n, p, ranks, D, U, V, R, W, B, c=None) -> np.ndarray:
    c = _tree(n, p, c)
    ranks = np.ascontiguousarray(ranks if p > 0 else [0], dtype=np.int32)
    D, U, V, R, W, B = (_f64(a) for a in (D, U, V, R, W, B))
    A = np.empty((n, n), dtype=np.float64)
    rc = _load().oracle_hss_dense_ranked(n, p, _ptr(c), _ptr(ranks), _ptr(D), _ptr(U), _ptr(V), _ptr(R), _ptr(W),
                                         _ptr(B), _ptr(A))
    _check(rc, "hss_dense_ranked")
    return A


def hss_matvec_noderanked(n, p, node_ranks, D, U, V, R, W, B, X, c=None, trans=False) -> np.ndarray:
    """Y = A X (A^T X if trans) for an HSS matrix with per-node ranks, node (l, i)
    at heap index 2^l - 2 + i; layout in hm_oracle.h."""
    c = _tree(n, p, c)
    X = _X2(X)
    m = X.shape[1]
    nr = np.ascontiguousarray(node_ranks if p > 0 else [0], dtype=np.int32)
    D, U, V, R, W, B = (_f64(a) for a in (D, U, V, R, W, B))
    Y = np.empty((n, m), dtype=np.float64)
    fn = _load().oracle_hss_matvec_noderanked_t if trans else _load().oracle_hss_matvec_noderanked
    rc = fn(n, p, _ptr(c), _ptr(nr), _ptr(D), _ptr(U), _ptr(V), _ptr(R), _ptr(W), _ptr(B), _ptr(X), m, _ptr(Y))
    _check(rc, "hss_matvec_noderanked")
    return Y


def hss_dense_noderanked(n, p, node_ranks, D, U, V, R, W, B, c=None) -> np.ndarray:
    c = _tree(n, p, c)
    nr = np.ascontiguousarray(node_ranks if p > 0 else [0], dtype=np.int32)
    D, U, V, R, W, B = (_f64(a) for a in (D, U, V, R, W, B))
    A = np.empty((n, n), dtype=np.float64)
    rc = _load().oracle_hss_dense_noderanked(n, p, _ptr(c), _ptr(nr), _ptr(D), _ptr(U), _ptr(V), _ptr(R), _ptr(W),
                                             _ptr(B), _ptr(A))
    _check(rc, "hss_dense_noderanked")
    return A


def hodlr_dense(n, p, ranks, D, U, V, c=None) -> np.ndarray:
    c = _tree(n, p, c)
    ranks = np.ascontiguousarray(ranks if p > 0 else [0], dtype=np.int32)
    D, U, V = _f64(D), _f64(U), _f64(V)
    A = np.empty((n, n), dtype=np.float64)
    _check(_load().oracle_hodlr_dense(n, p, _ptr(c), _ptr(ranks), _ptr(D), _ptr(U), _ptr(V), _ptr(A)), "hodlr_dense")
    return A


def hss_dense(n, p, k, D, U, V, R, W, B, c=None) -> np.ndarray:
    c = _tree(n, p, c)
    D, U, V, R, W, B = (_f64(a) for a in (D, U, V, R, W, B))
    A = np.empty((n, n), dtype=np.float64)
    rc = _load().oracle_hss_dense(n, p, _ptr(c), k, _ptr(D), _ptr(U), _ptr(V), _ptr(R), _ptr(W), _ptr(B), _ptr(A))
    _check(rc, "hss_dense")
    return A


def dense_matvec(A, X) -> np.ndarray:
    A = _f64(A)
    X = _X2(X)
    n, m = A.shape[0], X.shape[1]
    Y = np.empty((n, m), dtype=np.float64)
    _check(_load().oracle_dense_matvec(n, _ptr(A), _ptr(X), m, _ptr(Y)), "dense_matvec")
    return Y


def laplacian_inverse_apply(X) -> np.ndarray:
    X = _X2(X)
    n, m = X.shape
    Y = np.empty((n, m), dtype=np.float64)
    _check(_load().oracle_laplacian_inverse_apply(n, _ptr(X), m, _ptr(Y)), "laplacian_inverse_apply")
    return Y


# ------------------------------------------------------------ adjoint (f1) --

def hodlr_matvec_t(n, p, ranks, D, U, V, X, c=None) -> np.ndarray:
    """Y = A^* X (A^T: real), Fig. 5 left on the adjoint's generators."""
    c = _tree(n, p, c)
    X = _X2(X)
    m = X.shape[1]
    ranks = np.ascontiguousarray(ranks if p > 0 else [0], dtype=np.int32)
    D, U, V = _f64(D), _f64(U), _f64(V)
    Y = np.empty((n, m), dtype=np.float64)
    rc = _load().oracle_hodlr_matvec_t(n, p, _ptr(c), _ptr(ranks), _ptr(D), _ptr(U), _ptr(V), _ptr(X), m, _ptr(Y))
    _check(rc, "hodlr_matvec_t")
    return Y


def hodlr_matvec_t_leaves(n, p, ranks, Dsel, U, V, X, leaves, c=None) -> np.ndarray:
    c = _tree(n, p, c)
    X = _X2(X)
    m = X.shape[1]
    ranks = np.ascontiguousarray(ranks if p > 0 else [0], dtype=np.int32)
    leaves = np.ascontiguousarray(leaves, dtype=np.int64)
    rows = sum(int(c[L] - (c[L - 1] if L > 0 else 0)) for L in leaves)
    Dsel, U, V = _f64(Dsel), _f64(U), _f64(V)
    Y = np.empty((rows, m), dtype=np.float64)
    rc = _load().oracle_hodlr_matvec_t_leaves(
        n, p, _ptr(c), _ptr(ranks), _ptr(Dsel), _ptr(U), _ptr(V), _ptr(X), m, _ptr(leaves), leaves.size, _ptr(Y)
    )
    _check(rc, "hodlr_matvec_t_leaves")
    return Y


def hss_matvec_t(n, p, k, D, U, V, R, W, B, X, c=None) -> np.ndarray:
    """Y = A^* X, Fig. 5 right on the adjoint's generators."""
    c = _tree(n, p, c)
    X = _X2(X)
    m = X.shape[1]
    D, U, V, R, W, B = (_f64(a) for a in (D, U, V, R, W, B))
    Y = np.empty((n, m), dtype=np.float64)
    rc = _load().oracle_hss_matvec_t(
        n, p, _ptr(c), k, _ptr(D), _ptr(U), _ptr(V), _ptr(R), _ptr(W), _ptr(B), _ptr(X), m, _ptr(Y)
    )
    _check(rc, "hss_matvec_t")
    return Y


def hss_matvec_t_leaves(n, p, k, Dsel, U, V, R, W, B, X, leaves, c=None) -> np.ndarray:
    c = _tree(n, p, c)
    X = _X2(X)
    m = X.shape[1]
    leaves = np.ascontiguousarray(leaves, dtype=np.int64)
    rows = sum(int(c[L] - (c[L - 1] if L > 0 else 0)) for L in leaves)
    Dsel, U, V, R, W, B = (_f64(a) for a in (Dsel, U, V, R, W, B))
    Y = np.empty((rows, m), dtype=np.float64)
    rc = _load().oracle_hss_matvec_t_leaves(
        n, p, _ptr(c), k, _ptr(Dsel), _ptr(U), _ptr(V), _ptr(R), _ptr(W), _ptr(B), _ptr(X), m,
        _ptr(leaves), leaves.size, _ptr(Y)
    )
    _check(rc, "hss_matvec_t_leaves")
    return Y


# ------------------------------------------------------ norm estimate (f2) --

def hodlr_norm2_est(n, p, ranks, D, U, V, x0, iters, c=None) -> float:
    """||A||_2 estimate: power method on A A^* (P:1146), `iters` steps from x0."""
    c = _tree(n, p, c)
    ranks = np.ascontiguousarray(ranks if p > 0 else [0], dtype=np.int32)
    D, U, V, x0 = _f64(D), _f64(U), _f64(V), _f64(x0).ravel()
    est = ctypes.c_double(0.0)
    rc = _load().oracle_hodlr_norm2_est(n, p, _ptr(c), _ptr(ranks), _ptr(D), _ptr(U), _ptr(V), _ptr(x0),
                                        int(iters), ctypes.addressof(est))
    _check(rc, "hodlr_norm2_est")
    return est.value


def hss_norm2_est(n, p, k, D, U, V, R, W, B, x0, iters, c=None) -> float:
    c = _tree(n, p, c)
    D, U, V, R, W, B, x0 = (_f64(a) for a in (D, U, V, R, W, B, x0))
    est = ctypes.c_double(0.0)
    rc = _load().oracle_hss_norm2_est(n, p, _ptr(c), k, _ptr(D), _ptr(U), _ptr(V), _ptr(R), _ptr(W), _ptr(B),
                                      _ptr(x0.ravel()), int(iters), ctypes.addressof(est))
    _check(rc, "hss_norm2_est")
    return est.value


# ----------------------------------------------------------- hss2hodlr (f3) --

def hss_to_hodlr(n, p, k, U, V, R, W, B, c=None):
    """(Uh, Vh) level-major [p][n][k]: exact HODLR factors of the HSS matrix."""
    c = _tree(n, p, c)
    U, V, R, W, B = (_f64(a) for a in (U, V, R, W, B))
    Uh = np.zeros(max(p, 1) * n * k, dtype=np.float64)
    Vh = np.zeros(max(p, 1) * n * k, dtype=np.float64)
    rc = _load().oracle_hss_to_hodlr(n, p, _ptr(c), k, _ptr(U), _ptr(V), _ptr(R), _ptr(W), _ptr(B),
                                     _ptr(Uh), _ptr(Vh))
    _check(rc, "hss_to_hodlr")
    return Uh[: p * n * k], Vh[: p * n * k]
