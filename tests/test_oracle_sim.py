"""Pins for oracle.sim (alg1 driver) against an independent fp64 matrix trajectory."""
import random

import numpy as np
import pytest

from oracle import algebra as A
from oracle import schedule as S
from oracle import sim
from oracle.gg import GroupGenerator
from rp_inputs import gen


def _matrix_trajectory(n, N, steps, groups_of_t, lr=0.1):
    """X_t = (X_{t-1} - eta*G_t) * prod F^G  (P:495 with the SGD term first, alg1 order), fp64."""
    X = np.stack([gen.x0(w, N).astype(np.float64) for w in range(n)], axis=1)
    eta = float(np.float32(lr))
    for t in range(1, steps + 1):
        Gt = np.stack([gen.grad(w, t, N).astype(np.float64) for w in range(n)], axis=1)
        X = X - eta * Gt
        W = np.eye(n)
        for g in groups_of_t(t):
            W = W @ A.group_matrix(n, g)
        X = A.apply(X, W)
    return X


@pytest.mark.parametrize("rule,n,k,nodes,m", [("shift_k", 4, 2, None, None), ("shift_k", 8, 3, None, None),
                                              ("paper4", 8, None, 2, 4)])
def test_lockstep_static_matches_fp64_matrix_trajectory(rule, n, k, nodes, m):
    N, T = 2048, 100
    X, log = sim.run_lockstep(n, N, T, mode="static", rule=rule, k=k, nodes=nodes, m=m)
    ref = _matrix_trajectory(n, N, T, lambda t: S.groups_for(rule, t, n=n, k=k, nodes=nodes, m=m))
    got = np.stack([X[w] for w in range(n)], axis=1).astype(np.float64)
    scale = np.abs(ref).max()
    assert np.max(np.abs(got - ref)) <= 1e-6 * scale      # north-star tolerance, fp32 vs fp64
    assert len(log) == T


def test_lockstep_gd_partitions_and_matches_matrix():
    n, N, T, k = 8, 1024, 30, 3
    X, log = sim.run_lockstep(n, N, T, mode="gd", k=k, c_thres=4, seed_gd=3)
    for t, groups in log:
        sizes = sorted(len(g) for g in groups)
        assert sizes == [2, 3, 3]                           # 8 idle workers, k = 3
        assert sorted(w for g in groups for w in g) == list(range(n))
    by_t = {t: [g for g in gs if len(g) > 1] for t, gs in log}
    ref = _matrix_trajectory(n, N, T, lambda t: by_t[t])
    got = np.stack([X[w] for w in range(n)], axis=1).astype(np.float64)
    assert np.max(np.abs(got - ref)) <= 1e-6 * np.abs(ref).max()


def test_slice_equals_full_run():
    # the method is elementwise: simulating [lo, hi) reproduces that slice of a full run bitwise
    Xf, _ = sim.run_lockstep(4, 4096, 5, mode="static", rule="shift_k", k=2)
    Xs, _ = sim.run_lockstep(4, 4096, 5, mode="static", rule="shift_k", k=2, lo=1000, hi=1500)
    for w in range(4):
        assert np.array_equal(Xf[w][1000:1500], Xs[w])


def _async_events(n, k, c_thres, iters, seed):
    """A random asynchronous interleaving of the alg1 worker loop against the oracle GG."""
    rnd = random.Random(seed)
    gg = GroupGenerator(n, k, c_thres=c_thres, seed_gd=3)
    left = [iters] * n
    events = []
    while True:
        s = gg.s
        choices = [("req", w) for w in range(n) if left[w] > 0 and s.handed[w] == -1]
        choices += [("done", q) for q, mem in s.groups.items() if all(s.handed[x] == q for x in mem)]
        if not choices:
            break
        ev, a = rnd.choice(choices)
        if ev == "req":
            seq, mem = gg.req(a)
            events.append({"ev": "req", "w": a, "seq": seq, "members": list(mem)})
            if left[a] == 1:
                gg.retire(a)
                events.append({"ev": "retire", "w": a})
        else:
            mem = gg.done(a)
            events.append({"ev": "done", "seq": a})
            for x in mem:
                left[x] -= 1
    assert not any(left)
    return events


def test_replay_async_trace_against_fp64_group_sequence():
    n, k, N = 6, 3, 512
    events = _async_events(n, k, 2, 6, seed=11)
    X, steps = sim.replay_trace(events, n, N, k=k, c_thres=2, seed_gd=3)
    assert steps == [6] * n
    # independent fp64 replay: per completed group, members step with their own t, then average
    groups = {e["seq"]: e["members"] for e in events if e["ev"] == "req"}
    Y = {w: gen.x0(w, N).astype(np.float64) for w in range(n)}
    t_of = [0] * n
    eta = float(np.float32(0.1))
    for e in events:
        if e["ev"] == "done":
            mem = groups[e["seq"]]
            for w in mem:
                t_of[w] += 1
                Y[w] = Y[w] - eta * gen.grad(w, t_of[w], N).astype(np.float64)
            mean = sum(Y[w] for w in mem) / len(mem)
            for w in mem:
                Y[w] = mean.copy()
    for w in range(n):
        assert np.max(np.abs(X[w] - Y[w])) <= 1e-6 * max(np.abs(Y[w]).max(), 1)


def test_replay_rejects_forged_grant():
    events = _async_events(4, 2, 0, 2, seed=1)
    for e in events:
        if e["ev"] == "req":
            e["members"] = list(reversed(range(4)))[:2]
            break
    with pytest.raises(Exception):
        sim.replay_trace(events, 4, 64, k=2, c_thres=0, seed_gd=3)


def test_section_length_only_syncs_every_L_steps():
    # with section length L, steps t % L != 0 are SGD only
    X, log = sim.run_lockstep(4, 256, 8, mode="static", rule="shift_k", k=2, section_length=4)
    for t, groups in log:
        if t % 4:
            assert all(len(g) == 1 for g in groups)
        else:
            assert any(len(g) == 2 for g in groups)
    # L = 1 reproduces the plain run
    X1, _ = sim.run_lockstep(4, 256, 8, mode="static", rule="shift_k", k=2, section_length=1)
    X0, _ = sim.run_lockstep(4, 256, 8, mode="static", rule="shift_k", k=2)
    assert all(np.array_equal(X1[w], X0[w]) for w in range(4))


def test_momentum_run_matches_fp64_reference():
    # momentum + weight decay trajectory vs an independent fp64 loop
    n, N, T, mu, wd = 4, 512, 30, 0.9, 1e-4
    X, _ = sim.run_lockstep(n, N, T, mode="static", rule="shift_k", k=2, momentum=(mu, wd))
    eta = float(np.float32(0.1))
    mu64, wd64 = float(np.float32(mu)), float(np.float32(wd))
    Y = np.stack([gen.x0(w, N).astype(np.float64) for w in range(n)], axis=1)
    Vm = np.zeros_like(Y)
    for t in range(1, T + 1):
        Gt = np.stack([gen.grad(w, t, N).astype(np.float64) for w in range(n)], axis=1)
        Vm = mu64 * Vm + (Gt + wd64 * Y)
        Y = Y - eta * Vm
        W = np.eye(n)
        for g in S.shift_k(n, 2, t):
            W = W @ A.group_matrix(n, g)
        Y = A.apply(Y, W)
    got = np.stack([X[w] for w in range(n)], axis=1).astype(np.float64)
    assert np.max(np.abs(got - Y)) <= 2e-6 * np.abs(Y).max()
