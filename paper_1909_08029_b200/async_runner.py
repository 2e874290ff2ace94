"""Asynchronous driver: one host thread per local worker, dynamic Group Generation.

Each worker thread runs alg1 at its own pace, with no
global barrier:

  compute   synthetic compute time T_c: a host sleep ("adding ... times the normal
            iteration time of sleep"; reading R13; a slowed worker adds
            s * T_c), or rp_compute_delay on the worker's stream (device busy wait)
  Step 2    rp_step(w, g, lr)
  Step 3    rp_group_generate(w): Group Buffer head or a Global Division over the
            idle workers that pass the slowdown filter;
            or, with policy="random", the basic GG of §4.1 (random group, lock vector,
            pending queue: the request is retried while the group waits)
  Step 4    rp_preduce(w, G) + rp_barrier_free_wait(w) (host wait, group-local)

With several GPUs (one process each) the contexts share ONE Group Generator in
POSIX shared memory (RP_FLAG_SHARED_GG); cross-GPU groups launch in GG order.
PyTorch provides device memory, threads and the peer-record exchange only.
"""
import threading
import time

import torch

from . import rp
from .rp import Context, RP_FLAG_SHARED_GG

SEED_X = 1
SEED_G = 2


def _ceil_to(v, m):
    return (v + m - 1) // m * m


class AsyncRunner:
    def __init__(self, world, n_params, *, group_size, c_thres=4, seed_gd=3, n_gpus=1, rank=0, device=None,
                 lr=0.1, job_id=0, peer_group=None, trace_path=None, grad_mode="per_step", flags=0,
                 policy="gd", nvls=0):
        if grad_mode not in ("per_step", "resident"):
            raise ValueError("grad_mode must be 'per_step' or 'resident'")
        self.device = rank if device is None else device
        torch.cuda.set_device(self.device)
        if n_gpus > 1:
            flags |= RP_FLAG_SHARED_GG
        if policy == "random":          # §4.1 random GG (k = 2: AD-PSGD)
            flags |= rp.RP_FLAG_RANDOM_GG
        elif policy != "gd":
            raise ValueError("policy must be 'gd' or 'random'")
        self.world, self.n, self.lr, self.grad_mode = world, n_params, lr, grad_mode
        self.n_gpus, self.peer_group = n_gpus, peer_group
        self.ctx = Context(world, n_params, n_gpus=n_gpus, rank=rank, device=self.device, group_size=group_size,
                           c_thres=c_thres, seed_gd=seed_gd, flags=flags, job_id=job_id)
        self.local = self.ctx.local_workers()
        ld = _ceil_to(n_params, 64)
        dev = torch.device("cuda", self.device)
        self.X = torch.empty((len(self.local), ld), dtype=torch.float32, device=dev)
        self.G = torch.empty((len(self.local), ld), dtype=torch.float32, device=dev)
        self.streams = {}
        for w in self.local:
            self.ctx.bind_worker(w, self.x(w), self.g(w))
            self.streams[w] = self.ctx.worker_stream(w)
        if n_gpus > 1:
            self.ctx.peer_setup(peer_group)
            if nvls:   # groups spanning >= nvls GPUs reduce inside the NVSwitch (rp_nvls_enable)
                self.ctx.nvls_enable(nvls, peer_group)
        if trace_path:
            self.ctx.trace_open(trace_path)
        for w in self.local:
            rp.fill_xi(self.x(w), n_params, SEED_X, w, 0, 0, self.streams[w])
            if grad_mode == "resident":
                rp.fill_xi(self.g(w), n_params, SEED_G, w, 1, 0, self.streams[w])
        torch.cuda.synchronize(self.device)

    def x(self, w):
        return self.X[self.local.index(w), :self.n]

    def g(self, w):
        return self.G[self.local.index(w), :self.n]

    def run(self, *, steps=None, window_s=None, delay_ns=None, delay_mode="device", wait_timeout_us=600_000_000):
        """Run every local worker until it did `steps` steps, or until `window_s` seconds have
        passed (then one final step each). Returns {w: steps completed} (within the window).
        delay_mode: "host" sleeps delay_ns(w) on the worker's thread before each step, "device"
        enqueues an rp_compute_delay busy wait on the worker's stream."""
        if (steps is None) == (window_s is None):
            raise ValueError("give exactly one of steps / window_s")
        done = {w: 0 for w in self.local}
        errors = []
        t_end = time.perf_counter() + window_s if window_s is not None else None

        def loop(w):
            try:
                torch.cuda.set_device(self.device)
                s = self.streams[w]
                t = 0
                while True:
                    t += 1
                    final = (t == steps) if steps is not None else time.perf_counter() >= t_end
                    if delay_ns is not None:
                        if delay_mode == "host":
                            time.sleep(delay_ns(w) / 1e9)
                        else:
                            rp.compute_delay(s, delay_ns(w))
                    if self.grad_mode == "per_step":
                        rp.fill_xi(self.g(w), self.n, SEED_G, w, t, 0, s)
                    self.ctx.step(w, None, self.lr)
                    g = self.ctx.group_generate_wait(w)    # random GG: retry while pending
                    if final:
                        self.ctx.retire(w)
                    self.ctx.preduce(w, g)
                    self.ctx.barrier_free_wait(w, wait_timeout_us)
                    if t_end is None or time.perf_counter() <= t_end:
                        done[w] += 1
                    if final:
                        return
            except Exception as e:  # surfaced to the caller
                errors.append((w, repr(e)))

        threads = [threading.Thread(target=loop, args=(w,), daemon=True) for w in self.local]
        for th in threads:
            th.start()
        for th in threads:
            th.join()
        if errors:
            raise RuntimeError(f"worker threads failed: {errors}")
        return done

    def close(self):
        torch.cuda.synchronize(self.device)
        if self.n_gpus > 1:
            import torch.distributed as dist
            dist.barrier(group=self.peer_group)
        self.ctx.close()
