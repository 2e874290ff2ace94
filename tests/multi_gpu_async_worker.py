"""One rank of an asynchronous multi-GPU run (launched by tests/test_gpu_multi.py): one host thread
per local worker, ONE shared Group Generator (RP_FLAG_SHARED_GG), worker 0 slowed. The merged
decision traces of all ranks replay through the CPU oracle; local replicas must match bit for bit."""
import json
import os
import random
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import sim  # noqa: E402
from paper_1909_08029_b200.async_runner import AsyncRunner  # noqa: E402


def main():
    a = json.loads(sys.argv[1])
    dist.init_process_group("gloo")
    rank, ngpu = dist.get_rank(), dist.get_world_size()
    local_rank = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local_rank)
    job = [random.getrandbits(62) + 1 if rank == 0 else None]
    dist.broadcast_object_list(job, src=0)
    world = a["wpg"] * ngpu
    tdir = a["tmp"]
    r = AsyncRunner(world, a["n"], group_size=a["k"], c_thres=a["c_thres"], seed_gd=7, n_gpus=ngpu, rank=rank,
                    device=local_rank, job_id=job[0], trace_path=os.path.join(tdir, f"trace.{rank}"))
    slow_ns = int(a.get("slow_us", 2000) * 1000)
    done = r.run(steps=a["steps"], delay_ns=lambda w: slow_ns if w == 0 else 100_000)
    torch.cuda.synchronize()
    dist.barrier()
    st = r.ctx.stats()
    r.ctx.trace_open(os.devnull)          # flush + close this rank's trace file
    dist.barrier()
    events = []
    for q in range(ngpu):
        with open(os.path.join(tdir, f"trace.{q}")) as f:
            events += [json.loads(ln) for ln in f if ln.strip()]
    events.sort(key=lambda e: e["n"])
    ok = [e["n"] for e in events] == list(range(len(events)))
    X, t_of = sim.replay_trace(events, world, a["n"], k=a["k"], c_thres=a["c_thres"], seed_gd=7,
                               workers_per_gpu=a["wpg"])
    ok = ok and t_of == [a["steps"]] * world and all(v == a["steps"] for v in done.values())
    for w in r.local:
        got = r.x(w).cpu().numpy()
        if not np.array_equal(got.view(np.uint32), X[w].view(np.uint32)):
            print(f"rank {rank} worker {w}: differs from the oracle replay "
                  f"(max abs {np.max(np.abs(got - X[w]))})", flush=True)
            ok = False
    print(f"rank {rank}: {'OK' if ok else 'FAIL'} events={len(events)} cross_gpu_groups={st['cross_gpu_groups']} "
          f"gd_calls={st['gd_calls']}", flush=True)
    flag = torch.tensor([0 if ok else 1])
    dist.all_reduce(flag)
    r.close()
    dist.destroy_process_group()
    sys.exit(int(flag.item() != 0))


if __name__ == "__main__":
    main()
