"""librp host logic (static schedules, GB + GD + filter, protocol checks) vs the oracle, bit-exact.

Runs on a host-only context (n_gpus = 0): no GPU needed.
"""
import json
import random

import pytest

import paper_1909_08029_b200 as rp
from oracle import schedule as S
from oracle.gg import GroupGenerator


def _groups_from_group_of(group_of):
    by = {}
    for w, gi in enumerate(group_of):
        if gi >= 0:
            by.setdefault(gi, []).append(w)
    return sorted(tuple(v) for v in by.values())


@pytest.mark.parametrize("nodes,m", [(4, 4), (2, 2), (8, 2), (8, 1), (1, 4), (3, 4), (2, 8), (4, 16), (5, 3)])
def test_paper4_bit_exact(nodes, m):
    n = nodes * m
    with rp.Context(n, 1024, n_gpus=0, nodes=nodes, group_size=min(2, n)) as c:
        for t in range(0, 40):
            group_of, ng = c.schedule_static(rp.RP_SCHED_PAPER4, t)
            got = _groups_from_group_of(group_of)
            want = sorted(tuple(g) for g in S.paper4(nodes, m, t))
            assert got == want and ng == len(want), (t, got, want)


@pytest.mark.parametrize("n,k", [(4, 2), (8, 3), (16, 3), (16, 2), (8, 4), (5, 5), (64, 16), (7, 1)])
def test_shift_k_bit_exact(n, k):
    with rp.Context(n, 1024, n_gpus=0, group_size=k) as c:
        for t in range(0, 3 * k + 2):
            group_of, ng = c.schedule_static(rp.RP_SCHED_SHIFT_K, t)
            assert _groups_from_group_of(group_of) == sorted(tuple(g) for g in S.shift_k(n, k, t))


def test_schedule_static_worker_and_skips():
    with rp.Context(16, 1024, n_gpus=0, nodes=4, group_size=2) as c:
        g = c.schedule_static_worker(rp.RP_SCHED_PAPER4, 2, 2)   # W2 skips at 4k+2
        assert g.member_list() == [2] and g.seq < 0
        g = c.schedule_static_worker(rp.RP_SCHED_PAPER4, 4, 8)
        assert g.member_list() == [0, 4, 8, 12]
        g2 = c.schedule_static_worker(rp.RP_SCHED_PAPER4, 4, 12)
        assert g2.seq == g.seq                                     # same group, same id for every member


def test_schedule_rule_errors():
    with rp.Context(6, 1024, n_gpus=0, nodes=4, group_size=2) as c:
        with pytest.raises(rp.RPError) as e:
            c.schedule_static(rp.RP_SCHED_PAPER4, 0)            # 6 workers on 4 nodes
        assert e.value.status == rp.RP_EINVAL
        with pytest.raises(rp.RPError):
            c.schedule_static(99, 0)


@pytest.mark.parametrize("n,k,c_thres,seed", [(8, 3, 4, 3), (16, 3, 4, 7), (16, 2, 0, 1), (5, 4, 2, 99),
                                              (64, 16, 0, 5), (12, 5, 3, 2**63 + 11),
                                              (64, 3, 4, 3)])   # bench cfg2 at N = 8
def test_gg_lockstep_bit_exact(n, k, c_thres, seed):
    og = GroupGenerator(n, k, c_thres=c_thres, seed_gd=seed)
    with rp.Context(n, 1024, n_gpus=0, group_size=k, c_thres=c_thres, seed_gd=seed) as c:
        for _step in range(50):
            seqs = set()
            for w in range(n):
                g = c.group_generate(w)
                seq, members = og.req(w)
                assert (g.seq, tuple(g.member_list())) == (seq, members)
                seqs.add(seq)
            for s in sorted(seqs):
                c.gg_release(s)
                og.done(s)
        st = c.stats()
        assert st["gd_calls"] == og.gd_calls and st["max_gb_depth"] == 1


@pytest.mark.parametrize("n,k,c_thres,seed", [(8, 3, 2, 1), (16, 3, 4, 2), (6, 2, 1, 3), (16, 4, 0, 4)])
def test_gg_async_interleavings_bit_exact(n, k, c_thres, seed, tmp_path):
    """Random request/completion/retire interleavings drive the C GG and the oracle GG alike."""
    rnd = random.Random(seed)
    og = GroupGenerator(n, k, c_thres=c_thres, seed_gd=seed)
    left = [rnd.randint(3, 12) for _ in range(n)]
    trace = tmp_path / "trace.jsonl"
    with rp.Context(n, 1024, n_gpus=0, group_size=k, c_thres=c_thres, seed_gd=seed) as c:
        c.trace_open(trace)
        while True:
            s = og.s
            choices = [("req", w) for w in range(n) if left[w] > 0 and s.handed[w] == -1]
            choices += [("done", q) for q, mem in s.groups.items() if all(s.handed[x] == q for x in mem)]
            if not choices:
                break
            ev, a = rnd.choice(choices)
            if ev == "req":
                g = c.group_generate(a)
                seq, mem = og.req(a)
                assert (g.seq, tuple(g.member_list())) == (seq, mem)
                if left[a] == 1:
                    c.retire(a)
                    og.retire(a)
            else:
                c.gg_release(a)
                for x in og.done(a):
                    left[x] -= 1
        assert not any(left)
    events = [json.loads(ln) for ln in open(trace)]
    assert sum(e["ev"] == "req" for e in events) == sum(1 for e in og.trace if e[0] == "req")
    # the trace replays through the oracle GG grant by grant
    from oracle import sim
    sim.replay_trace(events, n, 16, k=k, c_thres=c_thres, seed_gd=seed)


def test_gg_protocol_errors():
    with rp.Context(4, 1024, n_gpus=0, group_size=2, c_thres=0, seed_gd=3) as c:
        g = c.group_generate(0)
        with pytest.raises(rp.RPError) as e:
            c.group_generate(0)                       # second request before completion
        assert e.value.status == rp.RP_ESTATE
        with pytest.raises(rp.RPError) as e:
            c.gg_release(g.seq)                       # partner never requested
        assert e.value.status == rp.RP_EPROTO
        with pytest.raises(rp.RPError) as e:
            c.gg_release(12345)
        assert e.value.status == rp.RP_EPROTO
        other = [w for w in range(4) if w not in g.member_list()]
        c.retire(other[0])                            # holds no handed group: retired now
        with pytest.raises(rp.RPError) as e:
            c.group_generate(other[0])
        assert e.value.status == rp.RP_ESTATE


@pytest.mark.parametrize("n,k,seed", [(8, 3, 1), (6, 2, 7), (16, 3, 3), (5, 4, 11)])
def test_random_gg_interleavings_bit_exact(n, k, seed, tmp_path):
    """The §4.1 random GG (lock vector + pending queue) in C++ vs the oracle, request by request."""
    from oracle.gg import RandomGroupGenerator
    rnd = random.Random(seed)
    og = RandomGroupGenerator(n, k, seed_gd=seed)
    left = [rnd.randint(2, 8) for _ in range(n)]
    arrived = {}
    trace = tmp_path / "trace.jsonl"
    with rp.Context(n, 1024, n_gpus=0, group_size=k, seed_gd=seed, flags=rp.RP_FLAG_RANDOM_GG) as c:
        c.trace_open(trace)
        for _ in range(100000):
            if not any(left):
                break
            full = [q for q, a in arrived.items() if a == set(og.groups[q])]
            ready = [w for w in range(n) if left[w] and og.handed[w] == -1]
            if full and (not ready or rnd.random() < 0.5):
                q = rnd.choice(full)
                c.gg_release(q)
                for m in og.done(q):
                    left[m] -= 1
                del arrived[q]
                continue
            w = rnd.choice(ready)
            st, seq, mem = og.req(w)
            if st == "pending":
                with pytest.raises(rp.RPError) as e:
                    c.group_generate(w)
                assert e.value.status == rp.RP_EAGAIN and e.value.group.seq == seq
                continue
            g = c.group_generate(w)
            assert (g.seq, tuple(g.member_list())) == (seq, mem)
            if left[w] == 1:
                c.retire(w)
                og.retire(w)
            arrived.setdefault(seq, set()).add(w)
        assert not any(left)
        st = c.stats()
        assert st["gg_pending"] == og.n_pending and st["gg_granted"] == og.n_granted
    events = [json.loads(ln) for ln in open(trace)]
    from oracle import sim
    sim.replay_trace(events, n, 16, k=k, c_thres=0, seed_gd=seed, policy="random")


@pytest.mark.parametrize("nodes,m,k,c_thres", [(4, 4, 3, 0), (2, 8, 3, 4), (8, 2, 2, 0), (1, 8, 3, 0), (3, 5, 4, 2),
                                            (8, 8, 3, 0)])   # bench cfg2ii at N = 8
def test_inter_intra_lockstep_bit_exact(nodes, m, k, c_thres):
    n = nodes * m
    og = GroupGenerator(n, k, c_thres=c_thres, seed_gd=9, nodes=nodes)
    with rp.Context(n, 1024, n_gpus=0, group_size=k, c_thres=c_thres, seed_gd=9, nodes=nodes,
                    flags=rp.RP_FLAG_INTER_INTRA) as c:
        for _step in range(24):
            seqs = set()
            got = c.group_generate_many(list(range(n)))
            for w in range(n):
                seq, members = og.req(w)
                assert (got[w].seq, tuple(got[w].member_list())) == (seq, members)
                seqs.add(seq)
            for s in sorted(seqs):
                c.gg_release(s)
                og.done(s)
        assert c.stats()["max_gb_depth"] == 2


def test_inter_intra_async_interleavings_bit_exact(tmp_path):
    rnd = random.Random(5)
    n, nodes, k = 12, 3, 3
    og = GroupGenerator(n, k, c_thres=3, seed_gd=4, nodes=nodes)
    left = [rnd.randint(2, 6) for _ in range(n)]
    trace = tmp_path / "trace.jsonl"
    with rp.Context(n, 1024, n_gpus=0, group_size=k, c_thres=3, seed_gd=4, nodes=nodes,
                    flags=rp.RP_FLAG_INTER_INTRA) as c:
        c.trace_open(trace)
        while True:
            s = og.s
            choices = [("req", w) for w in range(n)
                       if s.handed[w] == -1 and not (s.retired >> w) & 1 and (left[w] > 0 or s.gb[w])]
            choices += [("done", q) for q, mem in s.groups.items() if all(s.handed[x] == q for x in mem)]
            if not choices:
                break
            ev, a = rnd.choice(choices)
            if ev == "req":
                g = c.group_generate(a)
                seq, mem = og.req(a)
                assert (g.seq, tuple(g.member_list())) == (seq, mem)
                if left[a] <= 1 and s.gb[a] == [seq]:
                    c.retire(a)
                    og.retire(a)
            else:
                c.gg_release(a)
                for x in og.done(a):
                    left[x] = max(0, left[x] - 1)
        assert not any(left) and not og.s.groups
    events = [json.loads(ln) for ln in open(trace)]
    from oracle import sim
    sim.replay_trace(events, n, 16, k=k, c_thres=3, seed_gd=4, ii_nodes=nodes)


def test_bf16_context_rules():
    # reading R26: the dtype is validated up front (bf16 multi-GPU contexts are accepted;
    # without a device they fail with RP_ENODEV, not RP_EINVAL)
    with rp.Context(4, 1024, n_gpus=0, group_size=2, dtype="bf16") as c:
        assert c.dtype == "bf16"
    with pytest.raises(rp.RPError) as e:
        rp.Context(4, 1024, n_gpus=2, group_size=2, dtype="bf16")
    assert e.value.status == rp.RP_ENODEV
    cfg = rp.rp.rp_config(world=4, n_gpus=0, n_params=16, workers_per_gpu=4, group_size=2, dtype=7)
    with pytest.raises(rp.RPError) as e:
        rp.rp.rp_init(cfg)
    assert e.value.status == rp.RP_EINVAL
