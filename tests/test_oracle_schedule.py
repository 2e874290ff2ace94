"""Pins for oracle.schedule (§4.2 static scheduler)."""
import pytest

from oracle import schedule as S
from conftest import golden_lines


def _parse_paper4_golden():
    groups, skips = {}, {}
    for ln in golden_lines("paper4_4x4.txt"):
        head, _, body = ln.partition(":")
        if head.endswith("skip"):
            skips[int(head.split()[0])] = sorted(int(v) for v in body.split())
        else:
            groups[int(head)] = sorted(tuple(int(v) for v in g.split()) for g in body.split("|"))
    return groups, skips


def test_paper4_matches_printed_table_4x4():
    groups, skips = _parse_paper4_golden()
    for t in range(12):
        got = sorted(tuple(g) for g in S.paper4(4, 4, t))
        assert got == groups[t % 4], t
        covered = {w for g in got for w in g}
        assert sorted(set(range(16)) - covered) == skips[t % 4]


def test_paper4_printed_facts_p879():
    # "W0, W4, W8 and W12 ... in the same group in the (4k)-th iteration"
    assert [0, 4, 8, 12] in S.paper4(4, 4, 8)
    # "W2, W6, W10 and W14 do not participate in any group in the (4k+2)-th iteration"
    covered = {w for g in S.paper4(4, 4, 6) for w in g}
    assert not covered & {2, 6, 10, 14}
    # "the schedule is periodic with a cycle length of 4"
    for t in range(4):
        assert S.paper4(4, 4, t) == S.paper4(4, 4, t + 4) == S.paper4(4, 4, t + 400)


def test_shift_k_examples():
    assert S.shift_k(4, 2, 0) == [[0, 1], [2, 3]]
    assert S.shift_k(4, 2, 1) == [[0, 3], [1, 2]]
    assert S.shift_k(8, 3, 1) == [[0, 1, 7], [2, 3, 4], [5, 6]]
    g16 = S.shift_k(16, 3, 0)
    assert sorted(len(g) for g in g16) == [3] * 5   # worker 15 alone -> skip
    # one SHIFT_K(4,2) cycle averages all four workers exactly: P2 P1 = all-1/4
    from oracle.algebra import group_matrix
    import numpy as np
    P = np.eye(4)
    for t in (0, 1):
        for g in S.shift_k(4, 2, t):
            P = P @ group_matrix(4, g)
    assert np.allclose(P, np.full((4, 4), 0.25))


def _find(parent, a):
    while parent[a] != a:
        parent[a] = parent[parent[a]]
        a = parent[a]
    return a


def _check_rule(n, cycle, groups_of_t):
    """per-phase disjointness, every worker in a >=2-group once per cycle, union-find connectivity."""
    parent = list(range(n))
    in_some = set()
    for t in range(cycle):
        seen = set()
        for g in groups_of_t(t):
            assert len(g) >= 2 and len(set(g)) == len(g)
            assert all(0 <= w < n for w in g)
            assert not (seen & set(g)), f"conflict at t={t}: {g}"
            seen |= set(g)
            in_some |= set(g)
            for w in g[1:]:
                parent[_find(parent, w)] = _find(parent, g[0])
    assert in_some == set(range(n)), f"uncovered {set(range(n)) - in_some}"
    assert len({_find(parent, w) for w in range(n)}) == 1, "cycle graph not connected (P:659-661)"


@pytest.mark.parametrize("nodes", range(2, 9))
@pytest.mark.parametrize("m", range(2, 9))
def test_paper4_exhaustive_properties(nodes, m):
    if nodes * m > 64:
        pytest.skip("world > 64")
    _check_rule(nodes * m, 4, lambda t: S.paper4(nodes, m, t))


@pytest.mark.parametrize("n", range(2, 17))
def test_shift_k_exhaustive_properties(n):
    for k in range(2, n + 1):
        _check_rule(n, k, lambda t: S.shift_k(n, k, t))


def test_paper4_one_worker_per_node_and_one_node():
    # m = 1: phase 0 is the only sync (all nodes); nodes = 1: no cross-node groups
    assert S.paper4(8, 1, 0) == [list(range(8))]
    assert S.paper4(8, 1, 1) == [] and S.paper4(8, 1, 2) == []
    assert S.paper4(1, 4, 0) == [[2, 3]]
    assert S.paper4(1, 4, 2) == [[0, 3]]
