"""Lockstep driver of one GPU's workers through the public librp API.

One call of :meth:`LockstepRunner.step` is one training iteration of alg1
 for every local worker, in the engine's fast path:

  Step 2  synthetic gradient on the worker's stream (rp_fill_xi) + rp_step
  Step 3  rp_schedule_static_worker or rp_group_generate for every
          worker in ascending order (GB + GD; every rank runs the
          same deterministic GG)
  Step 4  rp_batch_begin / rp_preduce per local worker / rp_batch_end
          (all of this GPU's groups in one fused kernel launch)
  wait    rp_barrier_free_wait(RP_WAIT_DEVICE): stream-ordered, no host block

PyTorch supplies device memory only. Replicas are rows of one (wpg, ld)
fp32 tensor with a 64-element-aligned row stride ld (16-B aligned rows for
any n_params), gradients likewise.
"""
import torch

from . import rp
from .rp import Context, RP_SCHED_GG, RP_SCHED_PAPER4, RP_SCHED_SHIFT_K, RP_WAIT_DEVICE

SEED_X = 1   # x_w^0[j] = xi(1, w, 0, j)
SEED_G = 2   #                            g_w^t[j] = xi(2, w, t, j)

RULES = {"paper4": RP_SCHED_PAPER4, "shift_k": RP_SCHED_SHIFT_K}


def _ceil_to(v, m):
    return (v + m - 1) // m * m


class LockstepRunner:
    def __init__(self, world, n_params, *, mode, rule=None, group_size=2, n_gpus=1, rank=0, device=None,
                 lr=0.1, c_thres=4, seed_gd=3, nodes=0, grad_mode="per_step", flags=0, init=True,
                 peer_group=None, section_length=1, momentum=None, nvls=0, dtype="f32", emulate=False):
        if mode not in ("static", "gd"):
            raise ValueError("mode must be 'static' or 'gd'")
        if mode == "static" and rule not in RULES:
            raise ValueError("static mode needs rule 'paper4' or 'shift_k'")
        if grad_mode not in ("per_step", "resident"):
            raise ValueError("grad_mode must be 'per_step' or 'resident'")
        self.device = rank if device is None else device
        torch.cuda.set_device(self.device)
        self.mode, self.rule, self.lr, self.grad_mode = mode, rule, lr, grad_mode
        self.section_length = max(1, int(section_length))   # iterations between syncs
        self.momentum = momentum                              # (mu, weight_decay)
        self.world, self.n = world, n_params
        self.n_gpus, self.peer_group = n_gpus, peer_group
        self.dtype = dtype                                    # "bf16": bf16 replicas (reading R26)
        # emulate: n_gpus VIRTUAL GPUs on this one device, every worker driven by this process
        # (RP_FLAG_EMULATE; the cross-GPU kernel of every virtual GPU in one cooperative launch)
        self.emulate = bool(emulate)
        if self.emulate:
            flags |= rp.RP_FLAG_EMULATE
        self.ctx = Context(world, n_params, n_gpus=n_gpus, rank=rank, device=self.device,
                           group_size=group_size, c_thres=c_thres, nodes=nodes, seed_gd=seed_gd, flags=flags,
                           dtype=dtype)
        self.local = self.ctx.local_workers()
        self.ld = _ceil_to(n_params, 64)
        dev = torch.device("cuda", self.device)
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        self.X = torch.empty((len(self.local), self.ld), dtype=tdt, device=dev)
        self.G = torch.empty((len(self.local), self.ld), dtype=tdt, device=dev)
        # fp32 staging of the generated inputs, one row per worker (each used on its own stream)
        self._tmp = (torch.empty((len(self.local), n_params), dtype=torch.float32, device=dev)
                     if dtype == "bf16" else None)
        self.V = (torch.zeros((len(self.local), self.ld), dtype=torch.float32, device=dev)
                  if momentum is not None else None)
        self.streams = {}
        for i, w in enumerate(self.local):
            self.ctx.bind_worker(w, self.x(w), self.g(w))
            self.streams[w] = self.ctx.worker_stream(w)
        if n_gpus > 1 and not self.emulate:
            # map the peers' replicas + flag arrays (CUDA IPC records exchanged over
            # torch.distributed; the data path is the library's NVLink kernel)
            self.ctx.peer_setup(peer_group)
            if nvls:   # groups spanning >= nvls GPUs reduce inside the NVSwitch (rp_nvls_enable)
                self.ctx.nvls_enable(nvls, peer_group)
        self.t = 0
        if init:
            self.init_replicas()
        if grad_mode == "resident":
            for w in self.local:
                self._fill(self.g(w), SEED_G, w, 1)
        self.synchronize()

    # -- memory ----------------------------------------------------------------------
    def _row(self, w):
        return self.local.index(w)

    def x(self, w):
        return self.X[self._row(w), :self.n]

    def g(self, w):
        return self.G[self._row(w), :self.n]

    def v(self, w):
        return self.V[self._row(w), :self.n]

    def _fill(self, dst, seed, w, t):
        """Seeded synthetic input xi(seed, w, t) into dst on w's stream; bf16 destinations get
        the fp32 values rounded to nearest-even (input preparation, like the oracle's)."""
        if self.dtype == "f32":
            rp.fill_xi(dst, self.n, seed, w, t, 0, self.streams[w])
            return
        tmp = self._tmp[self._row(w)]
        rp.fill_xi(tmp, self.n, seed, w, t, 0, self.streams[w])
        with torch.cuda.stream(torch.cuda.ExternalStream(self.streams[w], device=self.device)):
            dst.copy_(tmp)

    def init_replicas(self):
        for w in self.local:
            self._fill(self.x(w), SEED_X, w, 0)
        self.t = 0

    def synchronize(self):
        torch.cuda.synchronize(self.device)

    # -- one lockstep step ---------------------------------------------------------------
    def groups_for_step(self, t):
        """Step 3 for every local worker; returns ({w: rp_group}, [seq of non-local GG groups])."""
        groups, foreign = {}, []
        if t % self.section_length != 0:       # no synchronization this step: SGD only
            for w in self.local:
                groups[w] = rp.rp_group.make(-(1 + t * self.world + w), [w])
            return groups, foreign
        if self.mode == "static":
            for w in self.local:
                groups[w] = self.ctx.schedule_static_worker(RULES[self.rule], t, w)
        else:
            local = set(self.local)
            seen = set()
            # same request order (ascending) on every rank: the replicated GG stays identical
            for w, g in zip(range(self.world), self.ctx.group_generate_many(list(range(self.world)))):
                if w in local:
                    groups[w] = g
                elif g.seq not in seen and not (set(g.member_list()) & local):
                    foreign.append(g.seq)
                seen.add(g.seq)
            foreign = sorted(set(foreign))
        return groups, foreign

    def step(self, grads=None):
        """One lockstep step; `grads` optionally maps w -> device tensor to use as g."""
        t = self.t + 1
        for w in self.local:
            g = grads[w] if grads is not None else None
            if grads is None and self.grad_mode == "per_step":
                self._fill(self.g(w), SEED_G, w, t)
            if self.momentum is not None:
                self.ctx.step_momentum(w, g, self.lr, self.momentum[0], self.momentum[1], self.v(w))
            else:
                self.ctx.step(w, g, self.lr)
        groups, foreign = self.groups_for_step(t)
        self.ctx.batch_begin()
        try:
            for w in self.local:
                self.ctx.preduce(w, groups[w])
        finally:
            self.ctx.batch_end()
        for w in self.local:
            self.ctx.barrier_free_wait(w, RP_WAIT_DEVICE)
        for seq in foreign:
            self.ctx.gg_release(seq)
        self.t = t
        return groups

    def run_native(self, steps):
        """`steps` lockstep steps in ONE library call (rp_lockstep_run: the same sequence of
        calls as step(), issued from C++), with the bound (resident) gradients, plain SGD."""
        if self.grad_mode != "resident" or self.momentum is not None:
            raise ValueError("run_native: resident gradients and plain SGD only")
        rule = RP_SCHED_GG if self.mode == "gd" else RULES[self.rule]
        self.ctx.lockstep_run(rule, self.t + 1, steps, self.lr, self.section_length)
        self.t += steps

    def run(self, steps):
        log = []
        for _ in range(steps):
            groups = self.step()
            log.append((self.t, sorted({tuple(g.member_list()) for g in groups.values()})))
        return log

    def close(self):
        self.synchronize()
        if self.n_gpus > 1 and not self.emulate:
            # every rank's last kernel has seen its peers finish reading; the barrier keeps a
            # rank from freeing replicas another rank still has mapped
            import torch.distributed as dist
            dist.barrier(group=self.peer_group)
        self.ctx.close()
