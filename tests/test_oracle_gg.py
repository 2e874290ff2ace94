"""Pins for oracle.gg: Group Buffer + Global Division + slowdown filter (§5)."""
from collections import Counter

import pytest

from oracle.gg import ConflictError, GGState, GroupGenerator, ProtocolError


def _clone(gg):
    s = gg.s
    c = GroupGenerator.__new__(GroupGenerator)
    c.s = GGState(n=s.n, k=s.k, c_thres=s.c_thres, rng=s.rng, seq=s.seq,
                  gb=[list(b) for b in s.gb], counters=list(s.counters), lock=s.lock,
                  retired=s.retired, retiring=s.retiring, handed=list(s.handed),
                  groups=dict(s.groups))
    c.trace = []
    c.gd_calls = gg.gd_calls
    c.nodes = gg.nodes
    c.head_rot = list(gg.head_rot)
    return c


def test_global_division_paper_example_4_workers():
    # fig:global_devision: 4 workers, empty GBs. The first request
    # (W0) creates two disjoint pairs; W3's later request is served from its GB
    # without another GD ("GG will directly provide the non-conflicting [W1,W3]").
    gg = GroupGenerator(4, 2, c_thres=0, seed_gd=3)
    seq0, g0 = gg.req(0)
    assert 0 in g0 and len(g0) == 2 and gg.gd_calls == 1
    other = tuple(sorted(set(range(4)) - set(g0)))
    assert gg.s.groups[1] == other                 # the second group of the same GD
    w = other[-1]
    seq1, g1 = gg.req(w)
    assert g1 == other and seq1 == 1 and gg.gd_calls == 1   # served from GB, no new GD
    assert not set(g0) & set(g1)


def test_gd_sizes_16_idle_k3():
    # 16 idle workers, k = 3 -> 3,3,3,3,3,1 (remainder group, reading R8)
    gg = GroupGenerator(16, 3, c_thres=0, seed_gd=3)
    gg.req(5)
    sizes = sorted(len(m) for m in gg.s.groups.values())
    assert sizes == [1, 3, 3, 3, 3, 3]
    assert 5 in gg.s.groups[0]
    cover = [w for m in gg.s.groups.values() for w in m]
    assert sorted(cover) == list(range(16))


def test_gd_no_candidates_gives_singleton():
    gg = GroupGenerator(3, 3, c_thres=0, seed_gd=3)
    gg.req(0)          # takes all three
    gg.req(1)
    gg.req(2)
    gg.done(0)
    gg.retire(1)
    gg.retire(2)
    assert gg.req(0)[1] == (0,)


def test_slowdown_filter_rule_p1189():
    # c = [10, 10, 3, 10], initiator 0, C_thres = 5: worker 2 is filtered (10 - 3 >= 5).
    gg = GroupGenerator(4, 4, c_thres=5, seed_gd=3)
    gg.s.counters = [9, 10, 3, 10]   # req(0) increments c_0 to 10
    _, g = gg.req(0)
    assert g == (0, 1, 3)
    assert gg.s.gb[2] == []
    # slow initiator: c_i - c_w < C_thres holds for everyone, nobody filtered
    gg2 = GroupGenerator(4, 4, c_thres=5, seed_gd=3)
    gg2.s.counters = [10, 10, 2, 10]
    assert gg2.req(2)[1] == (0, 1, 2, 3)


def test_filter_disabled_and_counter_semantics():
    gg = GroupGenerator(4, 4, c_thres=0, seed_gd=3)
    gg.s.counters = [100, 0, 0, 0]
    assert gg.req(0)[1] == (0, 1, 2, 3)
    assert gg.s.counters == [101, 0, 0, 0]   # incremented at request time (R10)


def test_protocol_errors():
    gg = GroupGenerator(4, 2, c_thres=0, seed_gd=3)
    seq, g = gg.req(0)
    with pytest.raises(ProtocolError):
        gg.req(0)                 # second request before its group completed
    with pytest.raises(ProtocolError):
        gg.done(seq)              # the partner never requested
    gg.retire(3)                  # 3 holds no handed group: retired at once
    with pytest.raises(ProtocolError):
        gg.req(3)
    with pytest.raises(ProtocolError):
        gg.req(99)


def test_membership_frequency_uniform():
    # GD draws a uniformly random partition: a given other worker shares the
    # initiator's group with probability (k-1)/(n-1) (= 2/7 for n=8, k=3).
    n, k, trials = 8, 3, 20000
    gg = GroupGenerator(n, k, c_thres=0, seed_gd=12345)
    cnt = Counter()
    for _ in range(trials):
        seq, g = gg.req(0)
        for v in g:
            if v != 0:
                cnt[v] += 1
        for w in range(1, n):     # everyone requests, then all complete
            gg.req(w)
        for s in sorted(gg.s.groups):
            gg.done(s)
    for v in range(1, n):
        assert abs(cnt[v] / trials - (k - 1) / (n - 1)) < 0.015


def _explore(n, k, c_thres, iters, use_retire=True, seed=3, nodes=0, depth_max=1):
    """DFS over every interleaving of request / completion events.

    Worker model (alg1 loop): compute -> request -> (all members requested) -> group
    completes -> next iteration. A worker keeps requesting while it has iterations left or
    groups queued in its GB (Inter-Intra queues two); it declares retirement (reading R19)
    with the request that takes the last group it will ever run.
    Returns (states, deadlocks, max_gb_depth).
    """
    start = GroupGenerator(n, k, c_thres=c_thres, seed_gd=seed, nodes=nodes)
    stack = [(start, tuple([iters] * n))]
    seen = set()
    deadlocks = 0
    max_depth = 0
    while stack:
        gg, left = stack.pop()
        key = (gg.s.key(), tuple(gg.head_rot), left)
        if key in seen:
            continue
        seen.add(key)
        s = gg.s
        max_depth = max(max_depth, gg.gb_depth())
        # groups at the head of all their members' GBs run concurrently: they must be disjoint
        active = [m for q, m in s.groups.items() if all(s.gb[w] and s.gb[w][0] == q for w in m)]
        held = Counter(w for m in active for w in m)
        assert all(c <= 1 for c in held.values())
        succ = []
        for w in range(n):
            # Inter-Intra queues two groups: a worker serves what is queued for it before it stops
            if s.handed[w] == -1 and not (s.retired >> w) & 1 and (left[w] > 0 or (nodes and s.gb[w])):
                c = _clone(gg)
                seq, g = c.req(w)                   # raises ConflictError on overlap
                assert w in g                       # initiator is in its group
                if use_retire and left[w] <= 1 and (not nodes or c.s.gb[w] == [seq]):
                    c.retire(w)
                succ.append((c, left))
        for seq, members in s.groups.items():
            if all(s.handed[m] == seq for m in members):
                c = _clone(gg)
                c.done(seq)
                nl = list(left)
                for m in members:
                    nl[m] = max(0, nl[m] - 1)
                succ.append((c, tuple(nl)))
        if not succ and (any(left) or s.groups):
            deadlocks += 1
        stack.extend(succ)
    return len(seen), deadlocks, max_depth


@pytest.mark.parametrize("n,k,c_thres,iters", [
    (4, 2, 0, 2), (4, 3, 0, 2), (5, 3, 0, 2), (5, 2, 1, 1), (6, 3, 2, 1), (6, 2, 0, 1),
    (6, 3, 0, 2), (7, 3, 0, 1), (8, 3, 0, 1), (8, 2, 2, 1), (8, 4, 0, 1),
])
def test_brute_force_interleavings(n, k, c_thres, iters):
    states, deadlocks, depth = _explore(n, k, c_thres, iters)
    assert states > 10
    assert deadlocks == 0          # with the retire rule (reading R19)
    assert depth <= 1              # GB depth <= 1 under GD


def test_brute_force_finds_deadlock_without_retire_rule():
    # negative control: without excluding finished workers, GD can assign a worker
    # that will never request again, and that group never completes.
    _, deadlocks, _ = _explore(4, 2, 0, 2, use_retire=False)
    assert deadlocks > 0


def test_conflict_detection_is_live():
    gg = GroupGenerator(4, 2, c_thres=0, seed_gd=3)
    gg.req(0)
    gg.s.gb[1] = []           # corrupt: pretend worker 1 is idle while its lock bit is held
    gg.s.gb[2] = []
    gg.s.gb[3] = []
    gg.s.gb[0] = []
    gg.s.handed[0] = -1
    with pytest.raises(ConflictError):
        gg.req(0)


def test_inter_intra_spec_example_2x2():
    # S:360 (hand trace of §5.2 at minimum scale): 2 nodes x 2 workers, heads {0, 2}:
    # Inter {0,2}, {1}, {3}; Intra {0,1}, {2,3}; every GB holds Inter then Intra.
    gg = GroupGenerator(4, 2, c_thres=0, seed_gd=3, nodes=2)
    seq, g = gg.req(0)
    groups = [gg.s.groups[q] for q in sorted(gg.s.groups)]
    assert sorted(groups[:3]) == [(0, 2), (1,), (3,)]
    assert groups[3:] == [(0, 1), (2, 3)]
    assert g == (0, 2)
    assert all(len(b) == 2 for b in gg.s.gb)


@pytest.mark.parametrize("nodes,m,k", [(4, 4, 3), (2, 8, 3), (8, 2, 2), (4, 4, 4)])
def test_inter_intra_structure_lockstep(nodes, m, k):
    # only Head Workers form cross-node groups, the rest is node-local; the
    # Intra phase is one group per node; heads rotate; lockstep steps alternate Inter / Intra.
    n = nodes * m
    gg = GroupGenerator(n, k, c_thres=0, seed_gd=5, nodes=nodes)
    heads_seen = [set() for _ in range(nodes)]
    for step in range(2 * m):
        seen = {}
        for w in range(n):
            seq, mem = gg.req(w)
            seen[seq] = mem
        groups = list(seen.values())
        assert sorted(w for g in groups for w in g) == list(range(n))      # a partition
        if step % 2 == 0:   # Inter
            cross = [g for g in groups if len({w // m for w in g}) > 1]
            for g in cross:
                assert len({w // m for w in g}) == len(g)                   # <= 1 worker per node
            for g in cross:
                for w in g:
                    heads_seen[w // m].add(w)
        else:               # Intra: exactly the node partitions
            assert sorted(groups) == [tuple(range(a * m, (a + 1) * m)) for a in range(nodes)]
        for s in sorted(seen):
            gg.done(s)
    assert gg.head_rot == [m] * nodes        # one division per two steps; heads rotate per node
    for a in range(nodes):
        assert heads_seen[a] <= set(range(a * m, (a + 1) * m))
    assert gg.gb_depth() == 0


@pytest.mark.parametrize("n,nodes,k,iters", [(4, 2, 2, 1), (4, 2, 3, 1), (6, 2, 2, 1), (6, 3, 2, 1)])
def test_inter_intra_brute_force(n, nodes, k, iters):
    states, deadlocks, depth = _explore(n, k, 0, iters, nodes=nodes)
    assert states > 10 and deadlocks == 0 and depth <= 2
