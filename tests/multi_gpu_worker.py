"""One rank of a multi-GPU parity run (launched by tests/test_gpu_multi.py through torchrun).

Each rank drives its GPU's workers through the public API (cross-GPU groups run the
NVLink peer kernel) and checks its local replicas against the CPU oracle bit for bit.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import sim  # noqa: E402
from paper_1909_08029_b200.runner import LockstepRunner  # noqa: E402


def main():
    # one JSON positional argument (torchrun would try to parse --options after the script)
    a = argparse.Namespace(**{"rule": None, "steps": 10, "sample": 0, "ii": False, **json.loads(sys.argv[1])})
    dist.init_process_group("gloo")
    rank, ngpu = dist.get_rank(), dist.get_world_size()
    local_rank = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local_rank)
    world = a.wpg * ngpu
    ii = bool(getattr(a, "ii", False))
    nodes = ngpu if (a.rule == "paper4" or ii) else 0
    import paper_1909_08029_b200 as rp
    mom = tuple(a.momentum) if getattr(a, "momentum", None) else None
    native = bool(getattr(a, "native", False))   # rp_lockstep_run with resident gradients
    r = LockstepRunner(world, a.n, mode=a.mode, rule=a.rule, group_size=a.k, n_gpus=ngpu, rank=rank,
                       device=local_rank, nodes=nodes, flags=rp.RP_FLAG_INTER_INTRA if ii else 0, momentum=mom,
                       grad_mode="resident" if native else "per_step",
                       section_length=getattr(a, "section_length", 1), nvls=getattr(a, "nvls", 0),
                       dtype=getattr(a, "dtype", "f32"))
    if native:
        r.run_native(a.steps)
        log = None
    else:
        log = r.run(a.steps)
    r.synchronize()
    slices = [(0, a.n)] if not a.sample else [(0, a.sample), (a.n // 2, a.n // 2 + a.sample),
                                               (a.n - a.sample, a.n)]
    ok = True
    for lo, hi in slices:
        X, olog = sim.run_lockstep(world, a.n, a.steps, mode=a.mode, rule=a.rule, k=a.k, nodes=nodes,
                                   m=(world // nodes if nodes else None), workers_per_gpu=a.wpg, lo=lo, hi=hi,
                                   ii_nodes=ngpu if ii else 0, momentum=mom,
                                   section_length=getattr(a, "section_length", 1), dtype=getattr(a, "dtype", "f32"),
                                   grad_step=1 if native else None)
        for w in r.local:
            got = r.x(w)[lo:hi].float().cpu().numpy()   # bf16 widens exactly
            if getattr(a, "tol", 0) and not np.array_equal(got.view(np.uint32), X[w].view(np.uint32)):
                # NVLS with kp >= 3: the switch's summation order (reading R25) -> north-star bound
                err = float(np.max(np.abs(got.astype(np.float64) - X[w])))
                scale = float(np.max(np.abs(X[w])))
                print(f"rank {rank} worker {w}: not bit-exact, max abs {err:.3e} vs bound {a.tol * scale:.3e}",
                      flush=True)
                ok = ok and err <= a.tol * scale
                continue
            if not np.array_equal(got.view(np.uint32), X[w].view(np.uint32)):
                bad = np.flatnonzero(got.view(np.uint32) != X[w].view(np.uint32))
                print(f"rank {rank} worker {w} slice [{lo},{hi}): {bad.size} elements differ, first {bad[:5]}, "
                      f"max abs {np.max(np.abs(got - X[w]))}", flush=True)
                ok = False
    mine = [g for _, gs in log for g in gs] if log is not None else None
    olocal = [tuple(g) for _, gs in olog for g in sorted(gs) if set(g) & set(r.local)]
    if mine is not None and sorted(mine) != sorted(olocal):
        print(f"rank {rank}: group assignments differ from the oracle", flush=True)
        ok = False
    st = r.ctx.stats()
    print(f"rank {rank}: {'OK' if ok else 'FAIL'} cross_gpu_groups={st['cross_gpu_groups']} "
          f"nvls_groups={st['nvls_groups']} launches={st['kernel_launches']}", flush=True)
    if getattr(a, "nvls", 0) and st["nvls_groups"] == 0 and st["cross_gpu_groups"] > 0:
        print(f"rank {rank}: NVLS enabled but no group took the NVLS path", flush=True)
        ok = False
    flag = torch.tensor([0 if ok else 1])
    dist.all_reduce(flag)
    r.close()
    dist.destroy_process_group()
    sys.exit(int(flag.item() != 0))


if __name__ == "__main__":
    main()
