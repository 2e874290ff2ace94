"""Pins for oracle.gg.RandomGroupGenerator: the basic GG of §4.1."""
from collections import Counter

import pytest

from oracle.gg import GroupGenerator, ProtocolError, RandomGroupGenerator


def test_paper_walkthrough_p712_745():
    # fig:gg_lock: W0 and W7 request; GG generates [0,4,5] for W0 and sets the lock bits;
    # W7's [4,5,7] conflicts on W4, W5 and waits in the pending queue; after [0,4,5]
    # acknowledges, [4,5,7] is granted.
    gg = RandomGroupGenerator(8, 3)
    st, s0, g0 = gg.req(0, members=(0, 4, 5))
    assert (st, g0) == ("ok", (0, 4, 5)) and gg.lock == (1 << 0) | (1 << 4) | (1 << 5)
    st, s1, g1 = gg.req(7, members=(4, 5, 7))
    assert (st, g1) == ("pending", (4, 5, 7)) and gg.pending == [s1]
    assert gg.req(7)[0] == "pending"                       # a retry keeps waiting
    assert gg.counters[7] == 1                             # retries are not new requests
    assert gg.req(4)[1:] == (s0, (0, 4, 5))                # members notified of their group
    assert gg.req(5)[1:] == (s0, (0, 4, 5))
    gg.done(s0)                                            # ack: release, rescan the queue
    assert gg.pending == [] and gg.lock == (1 << 4) | (1 << 5) | (1 << 7)
    assert gg.req(7) == ("ok", s1, (4, 5, 7))


def test_initiator_in_group_and_uniform_membership():
    n, k, trials = 8, 3, 20000
    gg = RandomGroupGenerator(n, k, seed_gd=99)
    cnt = Counter()
    for _ in range(trials):
        st, seq, g = gg.req(0)
        assert st == "ok" and 0 in g and len(g) == k
        for v in g:
            if v != 0:
                cnt[v] += 1
        for m in g:
            if m != 0:
                gg.req(m)
        gg.done(seq)
    for v in range(1, n):
        assert abs(cnt[v] / trials - (k - 1) / (n - 1)) < 0.015   # uniform draw


def test_protocol_errors():
    gg = RandomGroupGenerator(4, 2)
    st, seq, g = gg.req(0)
    with pytest.raises(ProtocolError):
        gg.req(0)
    with pytest.raises(ProtocolError):
        gg.done(seq)          # the partner never requested


def _explore(n, k, iters, seed=3):
    """All interleavings of request / retry / completion for the random GG."""
    start = RandomGroupGenerator(n, k, seed_gd=seed)
    import copy
    stack = [(start, tuple([iters] * n))]
    seen = set()
    deadlocks = 0
    while stack:
        gg, left = stack.pop()
        key = (gg.rng, gg.seq, gg.lock, gg.retired, gg.retiring, tuple(map(tuple, gg.inbox)), tuple(gg.pending),
               tuple(gg.pending_of), tuple(gg.waiting), tuple(gg.handed), tuple(sorted(gg.groups.items())), left)
        if key in seen:
            continue
        seen.add(key)
        granted = [s for s in gg.groups if s not in gg.pending]
        held = Counter(m for s in granted for m in gg.groups[s])
        assert all(c <= 1 for c in held.values())                  # atomicity
        assert all(len(b) <= 1 for b in gg.inbox)
        succ = []
        for w in range(n):
            if left[w] > 0 and gg.handed[w] == -1:
                c = copy.deepcopy(gg)
                st, seq, g = c.req(w)
                assert w in g
                if st == "ok" and left[w] == 1:
                    c.retire(w)
                succ.append((c, left))
        for seq in granted:
            if all(gg.handed[m] == seq for m in gg.groups[seq]):
                c = copy.deepcopy(gg)
                mem = c.done(seq)
                nl = list(left)
                for m in mem:
                    nl[m] -= 1
                succ.append((c, tuple(nl)))
        if not succ and (any(left) or gg.groups):
            deadlocks += 1
        stack.extend(succ)
    return len(seen), deadlocks


@pytest.mark.parametrize("n,k,iters", [(3, 2, 2), (4, 2, 1), (4, 3, 1), (5, 2, 1)])
def test_brute_force_random_gg(n, k, iters):
    states, deadlocks = _explore(n, k, iters)
    assert states > 10 and deadlocks == 0


def test_global_division_avoids_the_conflicts_random_gg_has():
    # §5.1 motivation: over a random asynchronous request stream, the random GG
    # serializes conflicting groups (pending queue), GB + GD never produces one.
    import random
    n, k, iters = 16, 3, 30

    def drive(gen, is_random, seed):
        rnd = random.Random(seed)
        left = [iters] * n
        arrived = {}                   # seq -> members that requested it
        for _ in range(200000):
            if not any(left):
                return True
            handed = gen.handed if is_random else gen.s.handed
            ready = [w for w in range(n) if left[w] and handed[w] == -1]
            full = [q for q, a in arrived.items() if a == set(members_of[q])]
            if full and (not ready or rnd.random() < 0.5):
                q = rnd.choice(full)
                gen.done(q)
                for m in members_of[q]:
                    left[m] -= 1
                del arrived[q]
                continue
            w = rnd.choice(ready)
            if is_random:
                st, q, mem = gen.req(w)
                if st == "pending":
                    continue
            else:
                q, mem = gen.req(w)
            if left[w] == 1:
                gen.retire(w)          # declared with the final request (reading R19)
            members_of[q] = mem
            arrived.setdefault(q, set()).add(w)
        return False

    members_of = {}
    rg = RandomGroupGenerator(n, k, seed_gd=1)
    assert drive(rg, True, 0)
    members_of = {}
    gd = GroupGenerator(n, k, c_thres=0, seed_gd=1)
    assert drive(gd, False, 0)
    assert rg.n_pending > 0            # random groups conflict and wait in the queue
    assert gd.gd_calls > 0             # GD: a conflict would raise ConflictError inside
