#!/usr/bin/env python3
"""Benchmark of the fused SGD + P-Reduce hot path (Ripples, arXiv 1909.08029) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload NAME]

One "step" is one lockstep training iteration of every worker (alg1, PAPER.md
P:582-603): group determination (GB + GD or a static rule) + the fused SGD +
P-Reduce kernel(s) for all groups, with parameter and gradient vectors resident
in HBM. Prints ONE JSON line (rank 0). Metric: worker-steps/s (BASELINE.json:
"P-Reduce GB/s vs NVLink/HBM roofline; worker-steps/sec at 1/2/4/8 B200");
P-Reduce GB/s and the roofline fraction ride along.

--impl reference times the CPU oracle (test infrastructure; the one other
place this file runs oracle/) on a bounded sample of the same workload.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_R50 = 25_557_032      # torchvision ResNet-50 parameter count (BASELINE configs[1..2])
N_VGG = 138_357_544     # torchvision VGG-16 parameter count (configs[3..4])
L2_BYTES = 126 * 2**20

# name -> workload (per GPU: wpg workers; world = wpg * n_gpus)
WORKLOADS = {
    "cfg1": dict(desc="configs[0]: 4 workers, 1M fp32, k=2, static SHIFT_K(4,2), 1 GPU",
                 wpg=4, n=1 << 20, k=2, mode="static", rule="shift_k"),
    "cfg2": dict(desc="configs[1]: 8 workers on 1 B200, ResNet-50-sized 25.6M fp32, k=3, GB+GD",
                 wpg=8, n=N_R50, k=3, mode="gd", rule=None),
}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock + throttle reasons polled through NVML every 5 ms during the timed region
    (the same counters `nvidia-smi --query-gpu=clocks.sm,clocks_event_reasons.*` reads)."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, device):
        self.device, self.samples, self.stop, self.th = device, [], threading.Event(), None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._sample()
            self.th = threading.Thread(target=self._loop, daemon=True)
            self.th.start()
        except Exception:  # no NVML: clocks reported as null
            self.th = None
        return self

    def _sample(self):
        nv = self.nv
        sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except AttributeError:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        self.samples.append((sm, r))

    def _loop(self):
        while not self.stop.wait(0.005):
            try:
                self._sample()
            except Exception:
                return

    def __exit__(self, *exc):
        if self.th:
            self._sample()
            self.stop.set()
            self.th.join(1)

    def summary(self):
        if not self.samples:
            return None
        reasons = sorted({name for _, r in self.samples for name, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "NVML, 5 ms polling"}


def init_dist(args):
    """torchrun launch: one rank per GPU (RANK / LOCAL_RANK / WORLD_SIZE from the env)."""
    world_size = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world_size != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world_size}")
    return rank, local_rank, world_size


# ------------------------------------------------------------------------------------------
# ours
# ------------------------------------------------------------------------------------------

def run_ours(args, wl):
    import torch
    import paper_1909_08029_b200 as rp
    from paper_1909_08029_b200.runner import LockstepRunner

    rank, local_rank, n_gpus = init_dist(args)
    if n_gpus > 1:
        raise SystemExit("multi-GPU bench not wired yet")
    torch.cuda.set_device(local_rank)
    wpg, n, k = wl["wpg"], wl["n"], wl["k"]
    world = wpg * n_gpus
    runner = LockstepRunner(world, n, mode=wl["mode"], rule=wl["rule"], group_size=k, n_gpus=n_gpus,
                            rank=rank, device=local_rank, grad_mode="resident", flags=rp.RP_FLAG_TIMING)
    for _ in range(args.warmup):
        runner.step()
    runner.synchronize()
    runner.ctx.timing_read()                              # drop warm-up launches
    s0 = torch.cuda.ExternalStream(runner.streams[runner.local[0]])   # every batch launches here
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st0 = runner.ctx.stats()
    with ClockSampler(local_rank) as clk:
        runner.synchronize()
        ev0.record(s0)
        for _ in range(args.steps):
            runner.step()
        ev1.record(s0)
        runner.synchronize()
    st1 = runner.ctx.stats()
    ms = ev0.elapsed_time(ev1)
    tim = runner.ctx.timing_read()
    bytes_step = (st1["bytes_hbm"] - st0["bytes_hbm"]) / args.steps
    launches = st1["kernel_launches"] - st0["kernel_launches"]
    value = world * args.steps / (ms / 1e3)
    peaks, peak_src = measured_peaks()
    kern_gbs = tim["bytes_hbm"] / (tim["total_ms"] / 1e3) / 1e9 if tim["total_ms"] > 0 else None
    traffic = traffic_from_profiles(args.workload)
    e2e = run_e2e(runner, args, torch)
    out = {
        "metric": "worker-steps/s (P-Reduce GB/s vs NVLink/HBM roofline; worker-steps/sec at 1/2/4/8 B200)",
        "value": round(value, 1),
        "unit": "worker-steps/s",
        "n_gpus": n_gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms / args.steps, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (counter-based xi generator; resident replicas + gradients)",
        "impl": "ours",
        "preduce_gbs": round(bytes_step * args.steps / (ms / 1e3) / 1e9, 1),
        "config": {"workload": args.workload, "desc": wl["desc"], "world": world, "workers_per_gpu": wpg,
                   "n_params": n, "group_size": k, "schedule": wl["rule"] or "GB+GD (lockstep, ascending requests)",
                   "lr": 0.1, "bytes_per_step": int(bytes_step),
                   "l2": ("inputs larger than L2" if bytes_step > L2_BYTES else
                          "working set fits in L2 (no flush): L2-resident number")},
        "roofline": {"bound": "hbm", "kernel": "preduce_multi_kernel (fused SGD + P-Reduce)",
                     "achieved": round(kern_gbs, 1) if kern_gbs else None, "peak": peaks["hbm_gbs"],
                     "peak_source": peak_src, "unit": "GB/s",
                     "frac": round(kern_gbs / peaks["hbm_gbs"], 4) if kern_gbs else None,
                     "traffic": traffic, "launches_per_step": launches / args.steps,
                     "kernel_ms_per_launch": round(tim["total_ms"] / max(tim["launches"], 1), 4),
                     "algorithmic_bytes_per_launch": int(tim["bytes_hbm"] / max(tim["launches"], 1))},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "e2e": e2e,
    }
    if rank == 0 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(wl, n_gpus, budget_s=args.cpu_budget)
    runner.close()
    if rank == 0:
        print(json.dumps(out), flush=True)


def run_e2e(runner, args, torch):
    """Same metric through the public API with host buffers: per step, h2d of every local worker's
    gradient from pinned host memory, the lockstep step, and a blocking d2h read of the step's
    result (the first 4 averaged parameters of every local worker)."""
    steps = max(1, min(args.steps, args.e2e_steps))
    n = runner.n
    host_g = [torch.empty(n, dtype=torch.float32, pin_memory=True) for _ in runner.local]
    for i, w in enumerate(runner.local):
        host_g[i].copy_(runner.g(w), non_blocking=False)
    host_out = torch.empty((len(runner.local), 4), dtype=torch.float32, pin_memory=True)
    runner.synchronize()
    streams = {w: torch.cuda.ExternalStream(runner.streams[w]) for w in runner.local}
    t0 = time.perf_counter()
    for _ in range(steps):
        for i, w in enumerate(runner.local):
            with torch.cuda.stream(streams[w]):
                runner.g(w).copy_(host_g[i], non_blocking=True)
        runner.step()
        for i, w in enumerate(runner.local):
            with torch.cuda.stream(streams[w]):
                host_out[i].copy_(runner.x(w)[:4], non_blocking=True)
        for w in runner.local:
            streams[w].synchronize()
    dt = time.perf_counter() - t0
    return {"value": round(len(runner.local) * runner.ctx.cfg.n_gpus * steps / dt, 1) if dt > 0 else None,
            "unit": "worker-steps/s", "steps": steps,
            "h2d_bytes_per_step": 4 * n * len(runner.local),
            "d2h_bytes_per_step": 16 * len(runner.local),
            "timer": "host wall clock around the public-API steps (includes pinned h2d/d2h)"}


def traffic_from_profiles(workload):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(workload)
    except (OSError, ValueError):
        return None


# ------------------------------------------------------------------------------------------
# CPU oracle (cpu_baseline leg and --impl reference)
# ------------------------------------------------------------------------------------------

def oracle_steps(wl, n_gpus, sample, steps):
    """Time `steps` lockstep steps of the oracle on elements [0, sample) of every replica, with
    resident gradients like the GPU leg. Returns seconds."""
    import numpy as np
    from oracle import schedule as S
    from oracle.gg import GroupGenerator
    from oracle.update import fused_group_update
    from rp_inputs import gen

    world = wl["wpg"] * n_gpus
    X = {w: gen.x0(w, wl["n"], 0, sample) for w in range(world)}
    G = {w: gen.grad(w, 1, wl["n"], 0, sample) for w in range(world)}
    gg = GroupGenerator(world, wl["k"], c_thres=4, seed_gd=3) if wl["mode"] == "gd" else None
    lr = np.float32(0.1)
    t0 = time.perf_counter()
    for t in range(1, steps + 1):
        if gg is not None:
            seen = {}
            for w in range(world):
                seq, mem = gg.req(w)
                seen[seq] = mem
            groups = [seen[s] for s in sorted(seen)]
            for s in sorted(seen):
                gg.done(s)
        else:
            groups = S.groups_for(wl["rule"], t, n=world, k=wl["k"])
            covered = {w for g in groups for w in g}
            groups = groups + [(w,) for w in range(world) if w not in covered]
        for g in groups:
            fused_group_update(X, {w: G[w] for w in g}, g, lr, wl["wpg"])
    return time.perf_counter() - t0


def cpu_baseline(wl, n_gpus, budget_s=15.0):
    """The oracle as it stands, one host core, bounded sample scaled to the full vector."""
    world = wl["wpg"] * n_gpus
    sample = min(wl["n"], 1 << 20)
    dt = oracle_steps(wl, n_gpus, sample, 1)                        # calibrate
    steps = max(1, min(50, int(budget_s / max(dt, 1e-6))))
    dt = oracle_steps(wl, n_gpus, sample, steps)
    value = world * steps / dt * (sample / wl["n"])
    return {"value": round(value, 3), "unit": "worker-steps/s", "cores": 1, "kind": "oracle",
            "sample": f"{world} workers x elements [0,{sample}) of {wl['n']}, {steps} steps, "
                      f"{dt:.1f} s; scaled by {sample}/{wl['n']}",
            "cpu": cpu_model()}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip() + f" ({os.cpu_count()} logical cores on host)"
    except OSError:
        pass
    return None


def run_reference(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_gpus = args.gpus
    world = wl["wpg"] * n_gpus
    sample = min(wl["n"], 1 << 18)
    for _ in range(args.warmup):
        oracle_steps(wl, n_gpus, sample, 1)
    dts = [oracle_steps(wl, n_gpus, sample, 1) for _ in range(args.steps)]
    dt = sum(dts)
    value = world * args.steps / dt * (sample / wl["n"])
    cb = {"value": round(value, 3), "unit": "worker-steps/s", "cores": 1, "kind": "oracle",
          "sample": f"each step: {world} workers x elements [0,{sample}) of {wl['n']}; scaled by {sample}/{wl['n']}",
          "cpu": cpu_model()}
    out = {"metric": "worker-steps/s (P-Reduce GB/s vs NVLink/HBM roofline; worker-steps/sec at 1/2/4/8 B200)",
           "value": cb["value"], "unit": "worker-steps/s", "n_gpus": n_gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3 * wl["n"] / sample, 3),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic", "impl": "reference",
           "config": {"workload": args.workload, "desc": wl["desc"], "world": world, "n_params": wl["n"],
                      "group_size": wl["k"]},
           "cpu_baseline": cb,
           "e2e": {"value": cb["value"], "unit": "worker-steps/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=None)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.workload is None:
        args.workload = "cfg2"
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
