"""Engine semantics on the GPU: collective contract, errors, group-local completion,
asynchronous Group Generation with trace replay through the oracle (needs a B200)."""
import json
import threading
import time

import numpy as np
import pytest
import torch

import paper_1909_08029_b200 as rp
from oracle import sim

pytestmark = pytest.mark.gpu


def _ctx(world, n, **kw):
    ctx = rp.Context(world, n, n_gpus=1, **kw)
    X = torch.empty((world, n), dtype=torch.float32, device="cuda")
    G = torch.empty((world, n), dtype=torch.float32, device="cuda")
    for w in range(world):
        rp.fill_xi(X[w], n, 1, w, 0, 0, 0)
        rp.fill_xi(G[w], n, 2, w, 1, 0, 0)
        ctx.bind_worker(w, X[w], G[w])
    torch.cuda.synchronize()
    return ctx, X, G


def _status(fn, *a):
    with pytest.raises(rp.RPError) as e:
        fn(*a)
    return e.value.status, str(e.value)


def test_protocol_errors():
    ctx, X, G = _ctx(4, 1024, group_size=2)
    g01 = rp.rp_group.make(-1, [0, 1])
    assert _status(ctx.preduce, 2, g01)[0] == rp.RP_EPROTO            # not a member
    ctx.preduce(0, g01)
    assert _status(ctx.preduce, 1, rp.rp_group.make(-1, [1, 2]))[0] == rp.RP_EPROTO   # members disagree
    assert _status(ctx.preduce, 0, g01)[0] == rp.RP_ESTATE            # arrived again before waiting
    assert _status(ctx.barrier_free_wait, 0, rp.RP_WAIT_DEVICE)[0] == rp.RP_ESTATE   # not launched
    st, msg = _status(ctx.barrier_free_wait, 0, 2000)                  # partner never arrives
    assert st == rp.RP_ETIMEOUT and "[1]" in msg
    ctx.preduce(1, g01)
    ctx.barrier_free_wait(0, 5_000_000)
    ctx.barrier_free_wait(1, rp.RP_WAIT_DEVICE)
    assert _status(ctx.barrier_free_wait, 1, 0)[0] == rp.RP_ESTATE     # no group any more
    ctx.step(2, None, 0.1)
    assert _status(ctx.step, 2, None, 0.1)[0] == rp.RP_ESTATE          # already staged
    assert _status(ctx.preduce, 3, rp.rp_group.make(-9, [3, 3]))[0] == rp.RP_EINVAL
    bad = torch.empty(1025, dtype=torch.float32, device="cuda")
    assert _status(ctx.bind_worker, 3, bad[1:], None)[0] == rp.RP_EINVAL   # misaligned
    ctx.close()


def test_gg_group_must_be_the_handed_one():
    ctx, X, G = _ctx(4, 256, group_size=2, c_thres=0)
    g = ctx.group_generate(0)
    forged = rp.rp_group.make(g.seq, [0, 3] if g.member_list() != [0, 3] else [0, 2])
    assert _status(ctx.preduce, 0, forged)[0] == rp.RP_EPROTO
    ctx.close()


def test_batch_defers_launch():
    ctx, X, G = _ctx(2, 4096, group_size=2)
    g = rp.rp_group.make(-1, [0, 1])
    ctx.batch_begin()
    ctx.preduce(0, g)
    ctx.preduce(1, g)
    assert _status(ctx.barrier_free_wait, 0, rp.RP_WAIT_DEVICE)[0] == rp.RP_ESTATE
    ctx.batch_end()
    ctx.barrier_free_wait(0, rp.RP_WAIT_DEVICE)
    ctx.barrier_free_wait(1, rp.RP_WAIT_DEVICE)
    torch.cuda.synchronize()
    assert torch.equal(X[0], X[1])
    ctx.close()


def test_timing_events():
    ctx, X, G = _ctx(3, 1 << 20, group_size=3, flags=rp.RP_FLAG_TIMING)
    g = rp.rp_group.make(-1, [0, 1, 2])
    for _ in range(3):
        for w in range(3):
            ctx.step(w, None, 0.1)
            ctx.preduce(w, g)
        for w in range(3):
            ctx.barrier_free_wait(w, rp.RP_WAIT_DEVICE)
    t = ctx.timing_read()
    assert t["launches"] == 3 and t["total_ms"] > 0 and t["bytes_hbm"] == 3 * 12 * 3 * (1 << 20)
    ctx.close()


def test_disjoint_groups_no_global_barrier():
    # group {0,1} completes and its members continue while {2,3} has a missing member
    ctx, X, G = _ctx(4, 1 << 16, group_size=2)
    ga, gb = rp.rp_group.make(-1, [0, 1]), rp.rp_group.make(-2, [2, 3])
    ctx.preduce(0, ga)
    ctx.preduce(2, gb)
    ctx.preduce(1, ga)
    ctx.barrier_free_wait(0, 5_000_000)
    ctx.barrier_free_wait(1, 5_000_000)
    assert _status(ctx.barrier_free_wait, 2, 1000)[0] == rp.RP_ETIMEOUT
    ctx.preduce(3, gb)
    ctx.barrier_free_wait(2, 5_000_000)
    ctx.barrier_free_wait(3, 5_000_000)
    ctx.close()


@pytest.mark.parametrize("slow,policy,k", [(1, "gd", 3), (5, "gd", 3), (2, "random", 3), (2, "random", 2)])
def test_async_gd_threads_replay_bit_exact(tmp_path, slow, policy, k):
    """cfg 5 semantics on one GPU: one host thread per worker, dynamic GG (GB + GD + filter, or the
    random GG of §4.1 with its pending queue; k = 2 is AD-PSGD), worker 0 slowed; the decision
    trace replays through the oracle to the same bits."""
    world, n, steps, c_thres = 8, 50_000, 12, 2
    flags = rp.RP_FLAG_RANDOM_GG if policy == "random" else 0
    ctx, X, G = _ctx(world, n, group_size=k, c_thres=c_thres, seed_gd=7, flags=flags)
    trace = tmp_path / "trace.jsonl"
    ctx.trace_open(trace)
    errors = []

    def worker(w):
        try:
            torch.cuda.set_device(0)
            s = ctx.worker_stream(w)
            for t in range(1, steps + 1):
                if w == 0:
                    time.sleep(0.002 * slow)                # heterogeneity injection
                rp.fill_xi(G[w], n, 2, w, t, 0, s)
                ctx.step(w, None, 0.1)
                g = ctx.group_generate_wait(w)
                if t == steps:
                    ctx.retire(w)
                ctx.preduce(w, g)
                ctx.barrier_free_wait(w, 60_000_000)
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append((w, repr(e)))

    threads = [threading.Thread(target=worker, args=(w,)) for w in range(world)]
    for th in threads:
        th.start()
    for th in threads:
        th.join(120)
    assert not errors, errors
    torch.cuda.synchronize()
    events = [json.loads(ln) for ln in open(trace)]
    Xo, t_of = sim.replay_trace(events, world, n, k=k, c_thres=c_thres, seed_gd=7, policy=policy)
    assert t_of == [steps] * world
    for w in range(world):
        assert np.array_equal(X[w].cpu().numpy().view(np.uint32), Xo[w].view(np.uint32)), w
    st = ctx.stats()
    if policy == "gd":
        assert st["max_gb_depth"] <= 1 and st["gd_calls"] >= 1
    else:
        assert st["gg_granted"] >= world * steps // k
    ctx.close()
