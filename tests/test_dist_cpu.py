"""Multi-rank host logic on CPU (gloo, world_size 2): the replicated Group Generator stays
identical on every rank in lockstep, peer records survive the exchange, and the lockstep
release of groups with no local member keeps the replicas in step."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world_size, port, wpg, k, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    import paper_1909_08029_b200 as rp
    n = world_size * wpg
    local = set(range(rank * wpg, (rank + 1) * wpg))
    log = []
    # host-only context: the same GG every rank replicates in a multi-GPU lockstep run
    with rp.Context(n, 1024, n_gpus=0, group_size=k, c_thres=4, seed_gd=11) as c:
        for _ in range(steps):
            groups = c.group_generate_many(list(range(n)))
            step = sorted({(g.seq, tuple(g.member_list())) for g in groups})
            log.append(step)
            # release: groups with local members first (as their waits would), then the rest
            mine = [s for s, m in step if set(m) & local]
            other = [s for s, m in step if not set(m) & local]
            for s in mine + other:
                c.gg_release(s)
    logs = [None] * world_size
    dist.all_gather_object(logs, log)
    # a peer record makes the round trip through the object exchange byte for byte
    rec = rp.rp_peer_info()
    rec.rank, rec.n_local, rec.first_worker = rank, wpg, rank * wpg
    rec.x_offset[0] = 4096 * (rank + 1)
    recs = [None] * world_size
    dist.all_gather_object(recs, bytes(rec))
    ok = all(lg == logs[0] for lg in logs)
    back = [rp.rp_peer_info.from_buffer_copy(b) for b in recs]
    ok = ok and [r.rank for r in back] == list(range(world_size)) and back[1].x_offset[0] == 8192
    dist.destroy_process_group()
    q.put((rank, ok, len(log)))


@pytest.mark.parametrize("wpg,k", [(4, 3), (1, 2), (8, 3)])
def test_replicated_gg_identical_across_ranks(wpg, k):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, wpg, k, 25, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res), res
    assert all(n == 25 for _, _, n in res)


def _shared_gg_rank(rank, world_size, port, job_id, n, k, c_thres, rounds, tdir, q):
    """Each process requests for its own workers, concurrently with the other process, against
    ONE Group Generator in shared memory; every group is released once, by the rank owning its
    lowest member. The merged trace must replay grant-for-grant through the oracle GG."""
    import random
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    import paper_1909_08029_b200 as rp
    wpg = n // world_size
    mine = list(range(rank * wpg, (rank + 1) * wpg))
    ok = True
    rnd = random.Random(rank + 17)
    c = rp.Context(n, 1024, n_gpus=0, rank=rank, group_size=k, c_thres=c_thres, seed_gd=5,
                   flags=rp.RP_FLAG_SHARED_GG, job_id=job_id)
    c.trace_open(os.path.join(tdir, f"trace.{rank}"))
    dist.barrier()
    for r in range(rounds):
        granted = {}
        for w in rnd.sample(mine, len(mine)):
            g = c.group_generate(w)
            ok = ok and w in g.member_list()
            granted[g.seq] = g.member_list()
            if r == rounds - 1:
                c.retire(w)
        dist.barrier()                      # every worker of the round has requested
        for seq, members in sorted(granted.items()):
            if min(members) in mine:
                c.gg_release(seq)
        dist.barrier()
    c.trace_open(os.devnull)
    dist.barrier()
    c.close()
    dist.destroy_process_group()
    q.put((rank, ok))


@pytest.mark.parametrize("n,k,c_thres", [(8, 3, 2), (12, 4, 0), (6, 2, 1)])
def test_shared_gg_two_processes_replay(n, k, c_thres, tmp_path):
    import json
    import random
    from oracle import sim
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    job = random.getrandbits(62) + 1
    procs = [ctx.Process(target=_shared_gg_rank, args=(r, 2, port, job, n, k, c_thres, 20, str(tmp_path), q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res)
    events = []
    for r in range(2):
        events += [json.loads(ln) for ln in open(tmp_path / f"trace.{r}") if ln.strip()]
    events.sort(key=lambda e: e["n"])
    assert [e["n"] for e in events] == list(range(len(events)))      # one global GG order
    assert sum(e["ev"] == "req" for e in events) == 20 * n
    sim.replay_trace(events, n, 8, k=k, c_thres=c_thres, seed_gd=5)   # raises on any differing grant
