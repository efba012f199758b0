"""Pins of the oracle's HSS product with per-level and per-node ranks (
P:264: the bases and translation operators need not have k columns "for every level and
node ... as long as the dimensions are compatible").

- brute force: the dense matrix assembled in numpy from the definition (P:250-259,
  eq. (3) with k_{l+1} x k_l translation blocks), times X;
- equal ranks: bit for bit the uniform-rank oracle;
- zero padding: the same operator written as a uniform-rank HSS matrix with
  K = max k_l, every generator zero-padded (an exact embedding);
- the adjoint against the transposed dense matrix; a rank-0 level cuts the
  nested bases above it (all higher off-diagonal blocks vanish);
- per-node ranks: the dense definition with (k_{2i} + k_{2i+1}) x k_h translations and
  k_{2q} x k_{2q+1} cores (ragged trees, rank-0 nodes), and per-node ranks that are equal
  within each level reproduce the per-level product bit for bit.
"""
import numpy as np
import pytest
import scipy.linalg

import hm_inputs
import oracle
from test_oracle import relerr, tree_sets


def rw_offsets(p, ranks):
    """Offsets (in doubles) of the R / W blocks of levels 1..p-1 and of the B blocks of the
    sibling levels 1..p (layout of oracle/hm_oracle.h)."""
    k = {l: ranks[l - 1] for l in range(1, p + 1)}
    rw, b = {}, {}
    o = 0
    for l in range(1, p):
        rw[l] = o
        o += (1 << l) * 2 * k[l + 1] * k[l]
    rw_total = o
    o = 0
    for l in range(1, p + 1):
        b[l] = o
        o += (1 << (l - 1)) * 2 * k[l] * k[l]
    return rw, rw_total, b, o


def random_hss_ranked(c, p, ranks, rng):
    n = int(c[-1])
    sizes = np.diff(np.concatenate([[0], c]))
    kp = ranks[p - 1] if p else 0
    _, rwt, _, bt = rw_offsets(p, ranks)
    D = rng.standard_normal(int((sizes ** 2).sum()))
    return (D, rng.standard_normal(n * kp), rng.standard_normal(n * kp), rng.standard_normal(rwt),
            rng.standard_normal(rwt), rng.standard_normal(bt))


def dense_hss_ranked_np(n, p, ranks, D, U, V, R, W, B, c):
    """A_rep: D_i on the diagonal; sibling blocks U_a^(l) S_ab V_b^(l)T with the level-l
    bases (k_l columns) rebuilt by eq. (3) from the k_{l+1}-column bases of the children."""
    A = np.zeros((n, n))
    off = 0
    for (lo, hi) in tree_sets(c, p, p):
        s = hi - lo
        A[lo:hi, lo:hi] = D[off: off + s * s].reshape(s, s)
        off += s * s
    if p == 0:
        return A
    k = {l: ranks[l - 1] for l in range(1, p + 1)}
    rw, _, bo, _ = rw_offsets(p, ranks)
    Ub = {p: [U.reshape(n, k[p])[lo:hi] for (lo, hi) in tree_sets(c, p, p)]}
    Vb = {p: [V.reshape(n, k[p])[lo:hi] for (lo, hi) in tree_sets(c, p, p)]}
    for l in range(p - 1, 0, -1):
        Ub[l], Vb[l] = [], []
        blk = 2 * k[l + 1] * k[l]
        for i in range(1 << l):
            Rn = R[rw[l] + i * blk: rw[l] + (i + 1) * blk].reshape(2 * k[l + 1], k[l])
            Wn = W[rw[l] + i * blk: rw[l] + (i + 1) * blk].reshape(2 * k[l + 1], k[l])
            Ub[l].append(scipy.linalg.block_diag(Ub[l + 1][2 * i], Ub[l + 1][2 * i + 1]) @ Rn)
            Vb[l].append(scipy.linalg.block_diag(Vb[l + 1][2 * i], Vb[l + 1][2 * i + 1]) @ Wn)
    for l in range(1, p + 1):
        sets = tree_sets(c, p, l)
        kk = k[l] * k[l]
        for q in range(1 << (l - 1)):
            base = bo[l] + q * 2 * kk
            S12 = B[base: base + kk].reshape(k[l], k[l])
            S21 = B[base + kk: base + 2 * kk].reshape(k[l], k[l])
            a, b = 2 * q, 2 * q + 1
            A[sets[a][0]:sets[a][1], sets[b][0]:sets[b][1]] = Ub[l][a] @ S12 @ Vb[l][b].T
            A[sets[b][0]:sets[b][1], sets[a][0]:sets[a][1]] = Ub[l][b] @ S21 @ Vb[l][a].T
    return A


def pad_to_uniform(n, p, ranks, U, V, R, W, B):
    """The same operator as a uniform-rank HSS with K = max k_l: zero-padded generators."""
    K = max(ranks)
    k = {l: ranks[l - 1] for l in range(1, p + 1)}
    rw, _, bo, _ = rw_offsets(p, ranks)
    Up = np.zeros((n, K))
    Up[:, :k[p]] = U.reshape(n, k[p])
    Vp = np.zeros((n, K))
    Vp[:, :k[p]] = V.reshape(n, k[p])
    nt, nb = max((1 << p) - 2, 0), (1 << p) - 1
    Rp, Wp, Bp = np.zeros((nt, 2 * K, K)), np.zeros((nt, 2 * K, K)), np.zeros((nb, 2, K, K))
    for l in range(1, p):
        blk = 2 * k[l + 1] * k[l]
        for i in range(1 << l):
            for src, dst in ((R, Rp), (W, Wp)):
                g = src[rw[l] + i * blk: rw[l] + (i + 1) * blk].reshape(2, k[l + 1], k[l])
                dst[(1 << l) - 2 + i, :k[l + 1], :k[l]] = g[0]
                dst[(1 << l) - 2 + i, K:K + k[l + 1], :k[l]] = g[1]
    for l in range(1, p + 1):
        kk = k[l] * k[l]
        for q in range(1 << (l - 1)):
            g = B[bo[l] + q * 2 * kk: bo[l] + (q + 1) * 2 * kk].reshape(2, k[l], k[l])
            Bp[(1 << (l - 1)) - 1 + q, :, :k[l], :k[l]] = g
    return K, Up.ravel(), Vp.ravel(), Rp.ravel(), Wp.ravel(), Bp.ravel()


CASES = [
    # endpoints c, p, ranks (level 1..p)
    (np.arange(1, 5) * 16, 2, [3, 5]),
    (np.arange(1, 9) * 12, 3, [2, 4, 6]),
    (np.arange(1, 9) * 12, 3, [6, 4, 2]),
    (np.array([3, 7, 7, 20, 26, 26, 31, 40]), 3, [1, 3, 2]),   # ragged, empty leaves
    (np.arange(1, 17) * 10, 4, [4, 0, 3, 5]),                  # a rank-0 level
    (np.arange(1, 3) * 20, 1, [5]),                            # p = 1
]


@pytest.mark.parametrize("c,p,ranks", CASES)
@pytest.mark.parametrize("m", [1, 3])
def test_ranked_hss_vs_dense_definition(c, p, ranks, m):
    rng = np.random.default_rng(7 + p + m)
    n = int(c[-1])
    D, U, V, R, W, B = random_hss_ranked(c, p, ranks, rng)
    X = rng.standard_normal((n, m))
    A = dense_hss_ranked_np(n, p, ranks, D, U, V, R, W, B, c)
    Y = oracle.hss_matvec_ranked(n, p, ranks, D, U, V, R, W, B, X, c=c)
    assert relerr(Y, A @ X) < 1e-13
    Yt = oracle.hss_matvec_ranked(n, p, ranks, D, U, V, R, W, B, X, c=c, trans=True)
    assert relerr(Yt, A.T @ X) < 1e-13
    Ad = oracle.hss_dense_ranked(n, p, ranks, D, U, V, R, W, B, c=c)
    assert relerr(Ad, A) < 1e-13


@pytest.mark.parametrize("c,p,ranks", CASES)
def test_ranked_hss_equals_zero_padded_uniform(c, p, ranks):
    rng = np.random.default_rng(11 + p)
    n = int(c[-1])
    D, U, V, R, W, B = random_hss_ranked(c, p, ranks, rng)
    X = rng.standard_normal((n, 2))
    K, Up, Vp, Rp, Wp, Bp = pad_to_uniform(n, p, ranks, U, V, R, W, B)
    Yu = oracle.hss_matvec(n, p, K, D, Up, Vp, Rp, Wp, Bp, X, c=c)
    Yr = oracle.hss_matvec_ranked(n, p, ranks, D, U, V, R, W, B, X, c=c)
    assert relerr(Yr, Yu) < 1e-14


def test_equal_ranks_bitwise_uniform():
    n, p, k = 1024, 4, 6
    s = hm_inputs.hss_random(n, p, k, cid=77)
    X = hm_inputs.rhs(n, 3, cid=77)
    Y1 = oracle.hss_matvec(n, p, k, s.D, s.U, s.V, s.R, s.W, s.B, X)
    Y2 = oracle.hss_matvec_ranked(n, p, [k] * p, s.D, s.U, s.V, s.R, s.W, s.B, X)
    assert np.array_equal(Y1, Y2)


def test_rank_zero_level_cuts_the_bases_above():
    """k_2 = 0: U^(2) has no columns, so U^(1) = blockdiag(U^(2)) R = 0 as well — only
    the leaf-level and level-3 sibling blocks and D remain."""
    c, p, ranks = np.arange(1, 9) * 8, 3, [3, 0, 4]
    rng = np.random.default_rng(5)
    n = int(c[-1])
    D, U, V, R, W, B = random_hss_ranked(c, p, ranks, rng)
    A = dense_hss_ranked_np(n, p, ranks, D, U, V, R, W, B, c)
    assert not A[:32, 32:].any() and not A[32:, :32].any()  # level-1 blocks vanish
    X = rng.standard_normal((n, 1))
    assert relerr(oracle.hss_matvec_ranked(n, p, ranks, D, U, V, R, W, B, X, c=c), A @ X) < 1e-13


# ---------------------------------------------------------- per-node ranks --
# node (l, i), l = 1..p, at heap index h = 2^l - 2 + i (layout of oracle/hm_oracle.h)

def node_layout(c, p, kn):
    """Offsets of the per-node layout: U/V per leaf, R/W per node (levels 1..p-1), B per
    parent (levels 0..p-1, heap order from the root)."""
    h = lambda l, i: (1 << l) - 2 + i  # noqa: E731
    sizes = np.diff(np.concatenate([[0], c]))
    uo, o = [], 0
    for i in range(1 << p):
        uo.append(o)
        o += int(sizes[i]) * kn[h(p, i)]
    rw, o = {}, 0
    for l in range(1, p):
        for i in range(1 << l):
            rw[(l, i)] = o
            o += (kn[h(l + 1, 2 * i)] + kn[h(l + 1, 2 * i + 1)]) * kn[h(l, i)]
    rwt = o
    bo, o = {}, 0
    for l in range(1, p + 1):
        for q in range(1 << (l - 1)):
            bo[(l, q)] = o
            o += 2 * kn[h(l, 2 * q)] * kn[h(l, 2 * q + 1)]
    return uo, rw, rwt, bo, o


def random_hss_noderanked(c, p, kn, rng):
    n = int(c[-1])
    sizes = np.diff(np.concatenate([[0], c]))
    uo, rw, rwt, bo, bt = node_layout(c, p, kn)
    nu = sum(int(sizes[i]) * kn[(1 << p) - 2 + i] for i in range(1 << p))
    D = rng.standard_normal(int((sizes ** 2).sum()))
    return (D, rng.standard_normal(nu), rng.standard_normal(nu), rng.standard_normal(rwt), rng.standard_normal(rwt),
            rng.standard_normal(bt))


def dense_hss_noderanked_np(n, p, kn, D, U, V, R, W, B, c):
    """A_rep from P:250-259 with per-node column counts: leaf bases |I_i| x k_h, U^(l) of
    node h = blockdiag(children) [Rl; Rr] ((k_{2i} + k_{2i+1}) x k_h), sibling blocks
    U_a S_ab V_b^T with S_{2q,2q+1}: k_{2q} x k_{2q+1}."""
    h = lambda l, i: (1 << l) - 2 + i  # noqa: E731
    A = np.zeros((n, n))
    off = 0
    for (lo, hi) in tree_sets(c, p, p):
        s = hi - lo
        A[lo:hi, lo:hi] = D[off: off + s * s].reshape(s, s)
        off += s * s
    if p == 0:
        return A
    uo, rw, _, bo, _ = node_layout(c, p, kn)
    Ub, Vb = {}, {}
    for i, (lo, hi) in enumerate(tree_sets(c, p, p)):
        k = kn[h(p, i)]
        Ub[(p, i)] = U[uo[i]: uo[i] + (hi - lo) * k].reshape(hi - lo, k)
        Vb[(p, i)] = V[uo[i]: uo[i] + (hi - lo) * k].reshape(hi - lo, k)
    for l in range(p - 1, 0, -1):
        for i in range(1 << l):
            k, k0, k1 = kn[h(l, i)], kn[h(l + 1, 2 * i)], kn[h(l + 1, 2 * i + 1)]
            Rn = R[rw[(l, i)]: rw[(l, i)] + (k0 + k1) * k].reshape(k0 + k1, k)
            Wn = W[rw[(l, i)]: rw[(l, i)] + (k0 + k1) * k].reshape(k0 + k1, k)
            Ub[(l, i)] = scipy.linalg.block_diag(Ub[(l + 1, 2 * i)], Ub[(l + 1, 2 * i + 1)]) @ Rn
            Vb[(l, i)] = scipy.linalg.block_diag(Vb[(l + 1, 2 * i)], Vb[(l + 1, 2 * i + 1)]) @ Wn
    for l in range(1, p + 1):
        sets = tree_sets(c, p, l)
        for q in range(1 << (l - 1)):
            a, b = 2 * q, 2 * q + 1
            k0, k1 = kn[h(l, a)], kn[h(l, b)]
            S12 = B[bo[(l, q)]: bo[(l, q)] + k0 * k1].reshape(k0, k1)
            S21 = B[bo[(l, q)] + k0 * k1: bo[(l, q)] + 2 * k0 * k1].reshape(k1, k0)
            A[sets[a][0]:sets[a][1], sets[b][0]:sets[b][1]] = Ub[(l, a)] @ S12 @ Vb[(l, b)].T
            A[sets[b][0]:sets[b][1], sets[a][0]:sets[a][1]] = Ub[(l, b)] @ S21 @ Vb[(l, a)].T
    return A


NODE_CASES = [
    (np.arange(1, 5) * 16, 2, [3, 5, 2, 4, 6, 1]),
    (np.arange(1, 9) * 12, 3, [2, 4, 6, 3, 1, 5, 2, 4, 3, 6, 1, 2, 5, 4]),
    (np.array([3, 7, 7, 20, 26, 26, 31, 40]), 3, [1, 3, 2, 0, 2, 1, 3, 2, 1, 0, 2, 3, 1, 2]),  # ragged, rank-0 nodes
    (np.arange(1, 3) * 20, 1, [5, 3]),
]


@pytest.mark.parametrize("c,p,kn", NODE_CASES)
def test_noderanked_hss_vs_dense_definition(c, p, kn):
    rng = np.random.default_rng(23 + p)
    n = int(c[-1])
    D, U, V, R, W, B = random_hss_noderanked(c, p, kn, rng)
    X = rng.standard_normal((n, 3))
    A = dense_hss_noderanked_np(n, p, kn, D, U, V, R, W, B, c)
    assert relerr(oracle.hss_matvec_noderanked(n, p, kn, D, U, V, R, W, B, X, c=c), A @ X) < 1e-13
    assert relerr(oracle.hss_matvec_noderanked(n, p, kn, D, U, V, R, W, B, X, c=c, trans=True), A.T @ X) < 1e-13
    assert relerr(oracle.hss_dense_noderanked(n, p, kn, D, U, V, R, W, B, c=c), A) < 1e-13


@pytest.mark.parametrize("c,p,ranks", CASES)
def test_noderanked_with_level_ranks_is_ranked(c, p, ranks):
    """Per-node ranks equal within each level are the per-level layout: bit for bit."""
    rng = np.random.default_rng(31 + p)
    n = int(c[-1])
    D, U, V, R, W, B = random_hss_ranked(c, p, ranks, rng)
    X = rng.standard_normal((n, 2))
    kn = [ranks[l - 1] for l in range(1, p + 1) for _ in range(1 << l)]
    assert np.array_equal(oracle.hss_matvec_noderanked(n, p, kn, D, U, V, R, W, B, X, c=c),
                          oracle.hss_matvec_ranked(n, p, ranks, D, U, V, R, W, B, X, c=c))
