"""Seeded synthetic inputs for the HODLR / HSS matvec (BASELINE.json configs 1-5).

This module serves BOTH sides — the oracle (tests) and the CUDA path (tests,
bench) — and therefore holds none of the method's arithmetic: it only draws
random generators with the shapes/distributions of DESIGN.md §4 and fills the
closed-form inverse-Laplacian generators (integer products plus one IEEE
division, bit-identical on any IEEE machine). It imports neither ``oracle``
nor ``paper_1909_07909_b200``.

Layouts (same as include/hm.h): row-major fp64;
  HODLR  D [2^p][b][b], U/V level-major [sum_l n*k_l] (level l = 1..p, [n][k_l]);
  HSS    D [2^p][b][b], U/V [n][k], R/W [2^p-2][2k][k], B [2^p-1][2][k][k].

Randomness: numpy's counter-based Philox bit generator, one independent stream
per (master seed, config id, array id, block id), so any block (a leaf, a row
slab of a level) can be drawn on its own — a rank can generate just its shard.
Array ids: X=0, D=1, U=2, V=3, R=4, W=5, B=6.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field
from typing import Dict, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_FILL_SRC = os.path.join(_HERE, "fill.c")
_FILL_LIB = os.path.join(_HERE, "libfill.so")
_fill = None


def build(force: bool = False) -> str:
    """Compile fill.c (the OpenMP host fill of the closed-form config-5 generators)."""
    if force or not os.path.exists(_FILL_LIB) or os.path.getmtime(_FILL_LIB) < os.path.getmtime(_FILL_SRC):
        tmp = _FILL_LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
                               "-Wall", "-o", tmp, _FILL_SRC])
        os.replace(tmp, _FILL_LIB)
    return _FILL_LIB


def _fill_lib():
    global _fill
    if _fill is None:
        lib = ctypes.CDLL(build())
        lib.fill_laplacian_leaves.argtypes = [ctypes.c_int64] * 4 + [ctypes.c_void_p]
        lib.fill_laplacian_leaves.restype = ctypes.c_int
        _fill = lib
    return _fill

MASTER_SEED = 190907909  # fixed and recorded in the bench output
AID = {"X": 0, "D": 1, "U": 2, "V": 3, "R": 4, "W": 5, "B": 6}


@dataclass(frozen=True)
class Config:
    """One BASELINE.json config (index 1..5), with the readings of DESIGN.md §3."""

    cid: int
    fmt: str  # "hodlr" | "hss"
    n: int
    leaf: int
    levels: int
    k: int
    nrhs: Tuple[int, ...]
    laplacian: bool = False
    gpus: Tuple[int, ...] = (1,)

    @property
    def nleaves(self) -> int:
        return 1 << self.levels


CONFIGS: Dict[int, Config] = {
    1: Config(1, "hodlr", 1024, 64, 4, 8, (1,)),
    2: Config(2, "hss", 4096, 64, 6, 16, (16,)),
    3: Config(3, "hodlr", 1 << 20, 256, 12, 16, (1, 8, 64)),
    4: Config(4, "hss", 1 << 22, 128, 15, 32, (32,), gpus=(1, 2, 4, 8)),
    5: Config(5, "hodlr", 1 << 24, 256, 16, 1, (1,), laplacian=True, gpus=(1, 2, 4, 8)),
}


def _rng(seed: int, cid: int, aid: int, block: int) -> np.random.Generator:
    key = np.array([(seed & 0xFFFFFFFF) | ((cid & 0xFFFF) << 32), (aid << 48) | (block & ((1 << 48) - 1))],
                   dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key))


def normal(shape, seed: int, cid: int, aid: int, block: int = 0) -> np.ndarray:
    """iid N(0,1) fp64 of the given shape from stream (seed, cid, aid, block)."""
    return _rng(seed, cid, aid, block).standard_normal(size=shape, dtype=np.float64)


def _orth_blocks(G: np.ndarray) -> np.ndarray:
    """Thin-QR Q factor of each block of a stack [N][r][k] (SURVEY G8/G10:
    'Gaussian orthonormalised (QR)'). Any Householder QR; Q is fixed once drawn.
    A block with fewer rows than columns (leaf b < rank k) gets orthonormal rows
    instead (Q of its transpose, transposed), keeping the [N][r][k] shape."""
    if G.shape[-2] < G.shape[-1]:
        q, _ = np.linalg.qr(np.swapaxes(G, -1, -2), mode="reduced")
        return np.ascontiguousarray(np.swapaxes(q, -1, -2))
    q, _ = np.linalg.qr(G, mode="reduced")
    return np.ascontiguousarray(q)


# ----------------------------------------------------------------- HODLR --

@dataclass
class Hodlr:
    n: int
    levels: int
    leaf: int
    ranks: np.ndarray  # int32 [levels]
    D: np.ndarray
    U: np.ndarray
    V: np.ndarray

    def level_slice(self, l: int) -> slice:
        off = int(self.n * int(self.ranks[: l - 1].sum()))
        return slice(off, off + self.n * int(self.ranks[l - 1]))


def hodlr_random(n: int, levels: int, ranks: Sequence[int], seed: int = MASTER_SEED, cid: int = 0,
                 rows: Optional[Tuple[int, int]] = None) -> Hodlr:
    """Random HODLR generators (configs 1 and 3; reading G7): D_i iid N(0,1)/sqrt(b),
    U_l, V_l iid N(0,1)/sqrt(s_l), s_l = n/2^l. If ``rows`` = (r0, r1) (aligned to
    leaves) only that row slab is drawn — a rank's shard; the full-array draw is the
    concatenation of the shards for any split."""
    b = n >> levels
    assert b << levels == n, "uniform tree: n = leaf * 2^levels"
    ranks = np.asarray(ranks if levels > 0 else [], dtype=np.int32).reshape(levels)
    r0, r1 = rows if rows is not None else (0, n)
    assert r0 % b == 0 and r1 % b == 0
    leaves = range(r0 // b, r1 // b)
    D = np.empty((len(leaves), b, b), dtype=np.float64)
    for t, i in enumerate(leaves):
        D[t] = normal((b, b), seed, cid, AID["D"], i) / np.sqrt(b)
    U = np.empty(((r1 - r0) * int(ranks.sum()),), dtype=np.float64)
    V = np.empty_like(U)
    off = 0
    for l in range(1, levels + 1):
        k = int(ranks[l - 1])
        s = n >> l
        # one stream per (level, leaf-sized slab) so shards are independent
        for name, dst in (("U", U), ("V", V)):
            blk = dst[off: off + (r1 - r0) * k].reshape(r1 - r0, k)
            for i in leaves:
                blk[(i * b - r0):(i * b - r0 + b)] = normal((b, k), seed, cid, AID[name], (l << 40) | i) / np.sqrt(s)
        off += (r1 - r0) * k
    return Hodlr(n, levels, b, ranks, D.reshape(-1), U, V)


def inverse_laplacian_leaf_blocks(n: int, levels: int, leaves=None, xp=np, device=None, chunk: int = 256):
    """D_i = A(I_i, I_i) of A = tridiag(-1,2,-1)^{-1}: A_ij = min(i,j)(n+1-max(i,j))/(n+1),
    1-based (BASELINE.json config 5). Integer product (< 2^53, exact) then one correctly
    rounded division: numpy and torch (CPU or CUDA) give identical bits. ``leaves``: list of
    leaf indices (default: all, in order). Filled ``chunk`` leaves at a time."""
    b = n >> levels
    assert b << levels == n
    kw = {} if xp is np else {"device": device}
    if leaves is None:
        leaves = range(1 << levels)
    if xp is np and isinstance(leaves, range) and leaves.step == 1:  # contiguous: the OpenMP fill
        out = np.empty(len(leaves) * b * b, dtype=np.float64)
        if _fill_lib().fill_laplacian_leaves(n, b, leaves.start, len(leaves), out.ctypes.data) != 0:
            raise ValueError("fill_laplacian_leaves: bad arguments")
        return out
    leaves = list(leaves)
    out = xp.empty((len(leaves), b, b), dtype=xp.float64, **kw)
    np1 = n + 1
    rr = xp.arange(1, b + 1, dtype=xp.int64, **kw)
    for a in range(0, len(leaves), chunk):
        sel = leaves[a:a + chunk]
        base = xp.asarray(np.asarray(sel, dtype=np.int64) * b) if xp is np else \
            xp.as_tensor(np.asarray(sel, dtype=np.int64) * b, device=device)
        g = base[:, None] + rr[None, :]               # 1-based global rows of each leaf
        gr, gc = g[:, :, None], g[:, None, :]
        mn = xp.minimum(gr, gc)
        mx = xp.maximum(gr, gc)
        num = mn * (np1 - mx)
        if xp is np:
            out[a:a + len(sel)] = num.astype(np.float64) / np1
        else:  # tensor / tensor: a true IEEE division (torch turns "/ scalar" into "* (1/scalar)")
            numf = num.to(xp.float64)
            out[a:a + len(sel)] = numf / xp.full_like(numf, float(np1))
    return out.reshape(-1)


def inverse_laplacian_factors(n: int, levels: int, xp=np, device=None, rows=None):
    """Level-major rank-1 factors (HODLR layout) of A = tridiag(-1,2,-1)^{-1} (reading G11):
    upper block (i<j): u_i = i, v_j = (n+1-j)/(n+1); lower block (i>j): u_i = n+1-i,
    v_j = j/(n+1). Row r of level l sits in node (r-1)//s_l; odd nodes are lower blocks.
    ``rows`` = (r0, r1): only those rows of every level (a rank's shard, same layout
    with r1 - r0 rows per level)."""
    kw = {} if xp is np else {"device": device}
    np1 = n + 1
    r0, r1 = rows if rows is not None else (0, n)
    nr = r1 - r0
    g = xp.arange(r0 + 1, r1 + 1, dtype=xp.int64, **kw)
    gf = g.astype(np.float64) if xp is np else g.to(xp.float64)
    # divisor as an array: torch turns "/ scalar" into "* (1/scalar)", which is not
    # correctly rounded; tensor / tensor is a true IEEE division like numpy's
    den = np1 if xp is np else xp.full_like(gf, float(np1))
    U = xp.empty(nr * levels, dtype=xp.float64, **kw)
    V = xp.empty(nr * levels, dtype=xp.float64, **kw)
    for l in range(1, levels + 1):
        s = n >> l
        odd = ((g - 1) // s) % 2 == 1
        U[(l - 1) * nr: l * nr] = xp.where(odd, np1 - gf, gf)
        V[(l - 1) * nr: l * nr] = xp.where(odd, (np1 - gf) / den, gf / den)
    return U, V


def hodlr_inverse_laplacian(n: int, levels: int, xp=np, device=None) -> Hodlr:
    """Exact HODLR form (rank 1 on every level) of tridiag(-1,2,-1)^{-1} (config 5)."""
    b = n >> levels
    D = inverse_laplacian_leaf_blocks(n, levels, xp=xp, device=device)
    U, V = inverse_laplacian_factors(n, levels, xp=xp, device=device)
    return Hodlr(n, levels, b, np.ones(levels, dtype=np.int32), D, U, V)


# ------------------------------------------------------------------- HSS --

@dataclass
class Hss:
    n: int
    levels: int
    leaf: int
    k: int
    D: np.ndarray
    U: np.ndarray
    V: np.ndarray
    R: np.ndarray
    W: np.ndarray
    B: np.ndarray


def hss_random(n: int, levels: int, k: int, seed: int = MASTER_SEED, cid: int = 0) -> Hss:
    """Random HSS generators (configs 2 and 4; readings G8/G10): leaf U_i, V_i (b x k)
    and R, W (2k x k) are thin-QR Q factors of Gaussian blocks; B12, B21 iid N(0,1);
    D_i iid N(0,1)/sqrt(b)."""
    b = n >> levels
    assert b << levels == n
    nl = 1 << levels
    D = np.empty((nl, b, b), dtype=np.float64)
    for i in range(nl):
        D[i] = normal((b, b), seed, cid, AID["D"], i) / np.sqrt(b)
    nt = max((1 << levels) - 2, 0)
    nb = (1 << levels) - 1
    if k > 0 and levels > 0:
        U = _orth_blocks(normal((nl, b, k), seed, cid, AID["U"]))
        V = _orth_blocks(normal((nl, b, k), seed, cid, AID["V"]))
        R = _orth_blocks(normal((nt, 2 * k, k), seed, cid, AID["R"])) if nt else np.zeros((0, 2 * k, k))
        W = _orth_blocks(normal((nt, 2 * k, k), seed, cid, AID["W"])) if nt else np.zeros((0, 2 * k, k))
        B = normal((nb, 2, k, k), seed, cid, AID["B"])
    else:
        U = np.zeros((nl, b, k)); V = np.zeros((nl, b, k))
        R = np.zeros((nt, 2 * k, k)); W = np.zeros((nt, 2 * k, k)); B = np.zeros((nb, 2, k, k))
    return Hss(n, levels, b, k, D.reshape(-1), U.reshape(-1), V.reshape(-1), R.reshape(-1), W.reshape(-1),
               B.reshape(-1))


def hss_inverse_laplacian(n: int, levels: int) -> Hss:
    """Exact rank-2 HSS form of tridiag(-1,2,-1)^{-1} (SURVEY §8(c) pins):
    U = [r, n+1-r] (1-based rows), V = U/(n+1), R = W = [I2; I2],
    B12 = [[0,1],[0,0]], B21 = [[0,0],[1,0]], D_i from the closed form."""
    b = n >> levels
    assert b << levels == n and levels >= 1
    D = inverse_laplacian_leaf_blocks(n, levels)
    g = np.arange(1, n + 1, dtype=np.float64)
    U = np.stack([g, (n + 1) - g], axis=1)
    V = U / (n + 1)
    nt, nb = (1 << levels) - 2, (1 << levels) - 1
    I2 = np.eye(2)
    R = np.tile(np.concatenate([I2, I2])[None], (nt, 1, 1))
    B = np.tile(np.array([[[0.0, 1.0], [0.0, 0.0]], [[0.0, 0.0], [1.0, 0.0]]])[None], (nb, 1, 1, 1))
    return Hss(n, levels, b, 2, D, U.reshape(-1), V.reshape(-1), R.reshape(-1), R.reshape(-1).copy(),
               B.reshape(-1))


def hss_random_ranked(n: int, levels: int, ranks: Sequence[int], seed: int = MASTER_SEED, cid: int = 0):
    """Random HSS generators with per-level ranks k_l = ranks[l-1] (the layout of
    include/hm.h hss_matvec_ranked): leaf U_i, V_i (b x k_p) and each node's R, W
    (2k_{l+1} x k_l) are thin-QR Q factors of Gaussian blocks (orthonormal rows when
    2k_{l+1} < k_l); cores N(0,1); D_i N(0,1)/sqrt(b). Returns an Hss with k = k_p and
    the flat level-major R, W, B of the ranked layout."""
    b = n >> levels
    assert b << levels == n and levels >= 1
    k = [int(r) for r in ranks]
    nl = 1 << levels
    D = np.empty((nl, b, b), dtype=np.float64)
    for i in range(nl):
        D[i] = normal((b, b), seed, cid, AID["D"], i) / np.sqrt(b)
    kp = k[-1]
    U = _orth_blocks(normal((nl, b, kp), seed, cid, AID["U"], 0)).reshape(-1) if kp else np.zeros(0)
    V = _orth_blocks(normal((nl, b, kp), seed, cid, AID["V"], 0)).reshape(-1) if kp else np.zeros(0)
    Rs, Ws, Bs = [], [], []
    for l in range(1, levels):
        kc, kl = k[l], k[l - 1]
        if kc and kl:
            Rs.append(_orth_blocks(normal((1 << l, 2 * kc, kl), seed, cid, AID["R"], l)).reshape(-1))
            Ws.append(_orth_blocks(normal((1 << l, 2 * kc, kl), seed, cid, AID["W"], l)).reshape(-1))
    for l in range(1, levels + 1):
        kl = k[l - 1]
        if kl:
            Bs.append(normal((1 << (l - 1)) * 2 * kl * kl, seed, cid, AID["B"], l))
    cat = lambda xs: np.concatenate(xs) if xs else np.zeros(0)  # noqa: E731
    return Hss(n, levels, b, kp, D.reshape(-1), U, V, cat(Rs), cat(Ws), cat(Bs))


def hss_random_noderanked(n: int, levels: int, node_ranks: Sequence[int], seed: int = MASTER_SEED,
                          cid: int = 0):
    """Random HSS generators with per-node ranks (include/hm.h
    hss_matvec_noderanked layout): node (l, i) has rank node_ranks[2^l - 2 + i]; leaf
    bases and translations are thin-QR Q factors of Gaussian blocks, cores N(0,1),
    D_i N(0,1)/sqrt(b). Returns an Hss (k = the largest leaf rank) with flat arrays."""
    b = n >> levels
    assert b << levels == n and levels >= 1
    kn = [int(r) for r in node_ranks]
    h = lambda l, i: (1 << l) - 2 + i  # noqa: E731
    nl = 1 << levels
    D = np.empty((nl, b, b), dtype=np.float64)
    for i in range(nl):
        D[i] = normal((b, b), seed, cid, AID["D"], i) / np.sqrt(b)
    Us, Vs, Rs, Ws, Bs = [], [], [], [], []
    for i in range(nl):
        k = kn[h(levels, i)]
        if k:
            Us.append(_orth_blocks(normal((1, b, k), seed, cid, AID["U"], i)).reshape(-1))
            Vs.append(_orth_blocks(normal((1, b, k), seed, cid, AID["V"], i)).reshape(-1))
    for l in range(1, levels):
        for i in range(1 << l):
            k, kc = kn[h(l, i)], kn[h(l + 1, 2 * i)] + kn[h(l + 1, 2 * i + 1)]
            if k and kc:
                Rs.append(_orth_blocks(normal((1, kc, k), seed, cid, AID["R"], h(l, i))).reshape(-1))
                Ws.append(_orth_blocks(normal((1, kc, k), seed, cid, AID["W"], h(l, i))).reshape(-1))
    for l in range(1, levels + 1):
        for q in range(1 << (l - 1)):
            cnt = 2 * kn[h(l, 2 * q)] * kn[h(l, 2 * q + 1)]
            if cnt:
                Bs.append(normal(cnt, seed, cid, AID["B"], h(l, 2 * q)))
    cat = lambda xs: np.concatenate(xs) if xs else np.zeros(0)  # noqa: E731
    return Hss(n, levels, b, max(kn[h(levels, i)] for i in range(nl)), D.reshape(-1), cat(Us), cat(Vs), cat(Rs),
               cat(Ws), cat(Bs))


def rhs(n: int, m: int, seed: int = MASTER_SEED, cid: int = 0, rows: Optional[Tuple[int, int]] = None,
        slab: int = 1 << 16) -> np.ndarray:
    """X iid N(0,1), [n][m], drawn in slabs of ``slab`` rows (shardable)."""
    r0, r1 = rows if rows is not None else (0, n)
    X = np.empty((r1 - r0, m), dtype=np.float64)
    s0 = r0 // slab
    for s in range(s0, (r1 + slab - 1) // slab):
        a, z = max(s * slab, r0), min((s + 1) * slab, r1)
        full = normal((slab, m), seed, cid, AID["X"], s)
        X[a - r0: z - r0] = full[a - s * slab: z - s * slab]
    return X


# ---------------------------------------------------------- device copies --

def device_hodlr_random(n, levels, ranks, seed, device, dtype=None):
    """Same distributions as hodlr_random, drawn with torch's device RNG (bench only:
    inputs resident in HBM without a host round trip; not bit-equal to the host draw)."""
    import torch
    b = n >> levels
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    D = torch.randn(n * b, dtype=torch.float64, device=device, generator=g).mul_(1.0 / np.sqrt(b))
    parts_u, parts_v = [], []
    for l in range(1, levels + 1):
        k = int(ranks[l - 1])
        s = n >> l
        parts_u.append(torch.randn(n * k, dtype=torch.float64, device=device, generator=g).mul_(1.0 / np.sqrt(s)))
        parts_v.append(torch.randn(n * k, dtype=torch.float64, device=device, generator=g).mul_(1.0 / np.sqrt(s)))
    U = torch.cat(parts_u) if parts_u else torch.zeros(0, dtype=torch.float64, device=device)
    V = torch.cat(parts_v) if parts_v else torch.zeros(0, dtype=torch.float64, device=device)
    return Hodlr(n, levels, b, np.asarray(ranks, dtype=np.int32), D, U, V)


def device_hss_random(n, levels, k, seed, device):
    """Same distributions as hss_random, drawn and orthonormalised on the device (bench only)."""
    import torch
    b = n >> levels
    nl = 1 << levels
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    f = dict(dtype=torch.float64, device=device, generator=g)
    D = torch.randn(nl * b * b, **f).mul_(1.0 / np.sqrt(b))
    nt, nb = (1 << levels) - 2, (1 << levels) - 1

    def orth(cnt, r):
        out = torch.empty(cnt, r, k, dtype=torch.float64, device=device)
        step = 8192
        for a in range(0, cnt, step):
            z = min(cnt, a + step)
            q, _ = torch.linalg.qr(torch.randn(z - a, r, k, **f), mode="reduced")
            out[a:z] = q
        return out.reshape(-1)

    U, V = orth(nl, b), orth(nl, b)
    R, W = orth(nt, 2 * k), orth(nt, 2 * k)
    B = torch.randn(nb * 2 * k * k, **f)
    return Hss(n, levels, b, k, D, U, V, R, W, B)


def device_hss_shard(n, levels, k, seed, device, P, r, block=64):
    """Rank r's shard (the dict of paper_1909_07909_b200.dist.hss_shard) of a device-drawn
    random HSS matrix with hss_random's distributions, drawing ONLY what the rank holds
    (bench only). Every array is drawn in blocks of `block` nodes, block j of (array,
    level) from its own seed, so the global matrix does not depend on P and a rank
    draws the blocks overlapping its nodes (the top levels' blocks on every rank)."""
    import torch
    b = n >> levels
    q = P.bit_length() - 1
    assert (1 << q) == P and q <= levels
    f = dict(dtype=torch.float64, device=device)

    def gen(aid, level, blk):
        g = torch.Generator(device=device)
        g.manual_seed((seed * 1000003 + aid * 10007 + level * 101) * 65537 + blk)
        return g

    def draw(aid, level, nodes, shape, lo, hi, orth=False, scale=1.0):
        """nodes [lo, hi) of the (aid, level) array of `nodes` nodes, each of `shape`."""
        out = []
        for blk in range(lo // block, (hi + block - 1) // block):
            a, z = blk * block, min(nodes, (blk + 1) * block)
            x = torch.randn(z - a, *shape, generator=gen(aid, level, blk), **f)
            if orth:
                x = torch.linalg.qr(x, mode="reduced")[0]
            out.append(x[max(lo, a) - a: min(hi, z) - a])
        x = torch.cat(out) if out else torch.empty(0, *shape, **f)
        return (x * scale if scale != 1.0 else x).reshape(-1)

    nl, lpr = 1 << levels, (1 << levels) // P
    L0, L1 = r * lpr, (r + 1) * lpr
    pl = levels - q
    sh = {"D": draw(AID["D"], levels, nl, (b, b), L0, L1, scale=1.0 / np.sqrt(b)),
          "U": draw(AID["U"], levels, nl, (b, k), L0, L1, orth=True),
          "V": draw(AID["V"], levels, nl, (b, k), L0, L1, orth=True)}
    tr = lambda aid, l, lo, hi: draw(aid, l, 1 << l, (2 * k, k), lo, hi, orth=True)  # noqa: E731
    cores = lambda l, lo, hi: draw(AID["B"], l, 1 << l, (2, k, k), lo, hi)  # noqa: E731
    cat = lambda xs: torch.cat(xs) if xs else torch.empty(0, **f)  # noqa: E731
    sh["W_sub"] = cat([tr(AID["W"], q + lp, r << lp, (r + 1) << lp) for lp in range(1, pl)])
    sh["R_sub"] = cat([tr(AID["R"], q + lp, r << lp, (r + 1) << lp) for lp in range(1, pl)])
    sh["B_sub"] = cat([cores(q + lp, r << lp, (r + 1) << lp) for lp in range(0, pl)])
    has_root = q >= 1 and pl >= 1
    sh["W_root"] = tr(AID["W"], q, r, r + 1) if has_root else torch.empty(0, **f)
    sh["R_root"] = tr(AID["R"], q, r, r + 1) if has_root else torch.empty(0, **f)
    sh["W_top"] = cat([tr(AID["W"], l, 0, 1 << l) for l in range(1, q)])
    sh["R_top"] = cat([tr(AID["R"], l, 0, 1 << l) for l in range(1, q)])
    sh["B_top"] = cat([cores(l, 0, 1 << l) for l in range(0, q)])
    return {key: v.contiguous() for key, v in sh.items()}
