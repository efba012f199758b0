"""The dataflow tree launch's schedule (csrc/hm_tree.cuh, hss_tree_flow_kernel) on the
host: tickets decode to pair tasks in dependency order, every flag a task waits for
is released by a task with a smaller ticket (so the launch cannot deadlock, whatever
the number of resident CTAs), every flag is released exactly once, and all indices
stay inside the workspace region the plan reserves (4 (1 + 2^(max(p, q) + 1))
bytes, csrc/hm_hss.cu). The decode below restates the kernel's formulas."""
import pytest


def decode(t, L, DL):
    """ticket -> ("up" | "down", level, pair) as in hss_tree_flow_kernel."""
    n_up = (1 << L) - 1 if L >= 1 else 0
    if t < n_up:
        v = (1 << L) - t  # in (2^(l-1), 2^l]
        l = (v - 1).bit_length()
        return "up", l, t - ((1 << L) - (1 << l))
    u = t - n_up
    l = (u + 1).bit_length()
    return "down", l, u + 1 - (1 << (l - 1))


def flags_of(kind, l, r, L):
    """(flags waited for, flag released), as indices into flags[] (0 = the ticket)."""
    upf = 1
    dnf = upf + (1 << L)
    if kind == "up":
        wait = [upf + (1 << l) - 1 + 2 * r, upf + (1 << l) - 1 + 2 * r + 1] if l + 1 <= L else []
        return wait, upf + (1 << (l - 1)) - 1 + r
    wait = []
    if l >= 2:
        wait.append(dnf + (1 << (l - 2)) - 1 + (r >> 1))
    if l <= L:
        wait.append(upf + (1 << (l - 1)) - 1 + r)
    return wait, dnf + (1 << (l - 1)) - 1 + r


@pytest.mark.parametrize("L,DL", [(0, 1), (1, 2), (3, 4), (5, 6), (9, 10), (10, 10), (0, 10), (7, 0), (14, 15)])
def test_schedule_invariants(L, DL):
    n_all = ((1 << L) - 1 if L >= 1 else 0) + ((1 << DL) - 1 if DL >= 1 else 0)
    released_by = {}
    seen = set()
    for t in range(n_all):
        kind, l, r = decode(t, L, DL)
        # a pair of level l exists: r < 2^(l-1)
        assert 1 <= l and 0 <= r < (1 << (l - 1)), (t, kind, l, r)
        assert (kind, l, r) not in seen
        seen.add((kind, l, r))
        wait, rel = flags_of(kind, l, r, L)
        for f in wait:
            assert f in released_by, (t, kind, l, r, f)  # released by an earlier ticket
        assert rel not in released_by  # released once
        released_by[rel] = t
    # every pair of every level in range was scheduled once
    assert len(seen) == n_all
    assert {(k, l) for k, l, _ in seen} == {("up", l) for l in range(1, L + 1)} | {("down", l) for l in range(1, DL + 1)}
    # indices inside the region the launch zeroes and the plan reserves
    used = max(released_by) + 1 if released_by else 1
    assert used <= 1 + (1 << L) + (1 << DL)
    p = max(L + 1, DL)
    assert 1 + (1 << L) + (1 << DL) <= 1 + (2 << p)


def test_up_children_and_down_parent():
    """Up pair (l, r) reads the child pairs (l+1, 2r), (l+1, 2r+1); down pair (l, q)
    reads its parent's pair (l-1, q >> 1) and the up pair (l, q) of its own x blocks."""
    L, DL = 4, 5
    order = {decode(t, L, DL): t for t in range(((1 << L) - 1) + ((1 << DL) - 1))}
    for (kind, l, r), t in order.items():
        if kind == "up" and l + 1 <= L:
            assert order[("up", l + 1, 2 * r)] < t and order[("up", l + 1, 2 * r + 1)] < t
        if kind == "down":
            if l >= 2:
                assert order[("down", l - 1, r >> 1)] < t
            if l <= L:
                assert order[("up", l, r)] < t
