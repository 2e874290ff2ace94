"""Watchdog check (launched by tests/test_gpu_multi.py through torchrun, 2 GPUs): rank 1 never
joins the cross-GPU group, so rank 0's kernel waits for its READY flag; with watchdog_s = 2 the
wait gives up, the kernel finishes and rank 0's host call reports RP_ETIMEOUT naming the flag
(round-1 advice: a fixed 30 s __trap killed the context instead)."""
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1909_08029_b200 as rp  # noqa: E402
from paper_1909_08029_b200.rp import Context, RPError, rp_group  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    torch.cuda.set_device(rank)
    n = 100_003
    ctx = Context(2, n, n_gpus=2, rank=rank, device=rank, group_size=2, watchdog_s=2)
    ld = (n + 63) // 64 * 64                 # 256-byte aligned rows, like the runner
    X = torch.zeros((2, ld), device="cuda")
    x, g = X[0, :n], X[1, :n]
    ctx.bind_worker(rank, x, g)
    ctx.peer_setup(None)
    ok = True
    if rank == 0:
        grp = rp_group.make(-1, [0, 1])
        ctx.step(0, None, 0.1)
        ctx.batch_begin()
        ctx.preduce(0, grp)
        ctx.batch_end()
        try:
            ctx.barrier_free_wait(0, 60_000_000)
            ok = False
            print("rank 0: no timeout reported", flush=True)
        except RPError as e:
            ok = e.status == rp.RP_ETIMEOUT and "timed out" in str(e)
            print(f"rank 0: {e}", flush=True)
        torch.cuda.synchronize()      # the context is still usable: no sticky error
    dist.barrier()
    print(f"rank {rank}: {'OK' if ok else 'FAIL'}", flush=True)
    flag = torch.tensor([0 if ok else 1])
    dist.all_reduce(flag)
    ctx.close()
    dist.destroy_process_group()
    sys.exit(int(flag.item() != 0))


if __name__ == "__main__":
    main()
