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

# NCCL's version banner would go to stdout ahead of the JSON line (NCCL_DEBUG=VERSION/INFO)
if not os.environ.get("RP_KEEP_NCCL_DEBUG"):
    os.environ["NCCL_DEBUG"] = "WARN"

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_R50 = 25_557_032      # torchvision ResNet-50 parameter count (BASELINE configs[1..2])
N_VGG = 138_357_544     # torchvision VGG-16 parameter count (configs[3..4])
L2_BYTES = 126 * 2**20

# name -> workload (per GPU: wpg workers; world = wpg * n_gpus)
WORKLOADS = {
    "cfg1": dict(desc="configs[0]: 4 workers, 1M fp32, k=2, static SHIFT_K(4,2), 1 GPU",
                 wpg=4, n=1 << 20, k=2, mode="static", rule="shift_k"),
    "cfg2": dict(desc="configs[1]: 8 workers per B200, ResNet-50-sized 25.6M fp32, k=3, GB+GD over all "
                      "8*N workers (N=1: exactly configs[1]; N>1: weak scaling of that layout)",
                 wpg=8, n=N_R50, k=3, mode="gd", rule=None),
    "cfg2ii": dict(desc="configs[1] layout (8 workers per B200, ResNet-50-sized, k=3) with Inter-Intra "
                        "Synchronization (§5.2, GPU = node): Head Workers across GPUs, the rest per GPU, "
                        "then whole-GPU groups",
                   wpg=8, n=N_R50, k=3, mode="gd", rule=None, inter_intra=True),
    "cfg2bf16": dict(desc="configs[1] layout (8 workers per B200, ResNet-50-sized, k=3, GB+GD) with bf16 replicas "
                          "and gradients, fp32 arithmetic, one rounding of the mean (SURVEY §8 f4, reading R26)",
                     wpg=8, n=N_R50, k=3, mode="gd", rule=None, dtype="bf16"),
    "cfg2iibf16": dict(desc="cfg2ii (Inter-Intra, 8 workers per B200, ResNet-50-sized, k=3) with bf16 replicas and "
                            "gradients: fp32 arithmetic, fp32 partials over NVLink, the mean rounded once to bf16",
                       wpg=8, n=N_R50, k=3, mode="gd", rule=None, inter_intra=True, dtype="bf16"),
    "cfg3": dict(desc="configs[2]: 1 worker per B200 (8 workers on 8 GPUs), ResNet-50-sized, k=3, GB+GD, "
                      "concurrent disjoint groups over NVLink",
                 wpg=1, n=N_R50, k=3, mode="gd", rule=None),
    "cfg4": dict(desc="configs[3]: 2 workers per B200 (16 on 8 GPUs), VGG-16-sized 138M fp32, k=3, static "
                      "SHIFT_K(2N,3)",
                 wpg=2, n=N_VGG, k=3, mode="static", rule="shift_k"),
    "xall": dict(desc="diagnostic: 1 worker per B200, ResNet-50-sized, ONE group of all N GPUs every step "
                      "(SHIFT_K(N,N)): the cross-GPU kernel's NVLink efficiency without lockstep skew",
                 wpg=1, n=N_R50, k=64, mode="static", rule="shift_k"),
    "xall_vgg": dict(desc="diagnostic: 1 worker per B200, VGG-16-sized, ONE group of all N GPUs every step",
                     wpg=1, n=N_VGG, k=64, mode="static", rule="shift_k"),
    "cfg5": dict(desc="configs[4]: 2 workers per B200, VGG-16-sized, k=3, asynchronous GB+GD+filter (C_thres=4), "
                      "worker 0 slowed by --slow x T_c of device delay per step (P:1395)",
                 wpg=2, n=N_VGG, k=3, mode="async", rule=None),
}
NVLINK_PEAK = 770.0   # GB/s per direction, measured peer copy (B200_PROFILING.md)
NVLINK_NOMINAL = 900.0
HBM_NOMINAL = 7700.0  # GB/s, B200 HGX HBM3e (B200_PROFILING.md)


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

def setup_dist(n_gpus, local_rank):
    """NCCL default group (plumbing + the NCCL baseline) and a gloo group for host metadata."""
    import torch
    import torch.distributed as dist
    if n_gpus == 1:
        return None
    dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    return dist.new_group(backend="gloo")


def max_over_ranks(v, pg):
    import torch
    import torch.distributed as dist
    if pg is None:
        return v
    t = torch.tensor([float(v)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=pg)
    return float(t.item())


def gather(obj, pg):
    import torch.distributed as dist
    if pg is None:
        return [obj]
    out = [None] * dist.get_world_size(pg)
    dist.all_gather_object(out, obj, group=pg)
    return out


def barrier(pg):
    import torch.distributed as dist
    if pg is not None:
        dist.barrier(group=pg)


def run_ours(args, wl):
    import torch
    import paper_1909_08029_b200 as rp
    from paper_1909_08029_b200.runner import LockstepRunner

    rank, local_rank, n_gpus = init_dist(args)
    torch.cuda.set_device(local_rank)
    pg = setup_dist(n_gpus, local_rank)
    wpg, n = wl["wpg"], wl["n"]
    world = wpg * n_gpus
    k = min(wl["k"], world)              # e.g. configs[2] at 2 GPUs: 2 workers, groups of 2
    flags = rp.RP_FLAG_TIMING | (rp.RP_FLAG_INTER_INTRA if wl.get("inter_intra") else 0)
    runner = LockstepRunner(world, n, mode=wl["mode"], rule=wl["rule"], group_size=k, n_gpus=n_gpus,
                            rank=rank, device=local_rank, grad_mode="resident", flags=flags,
                            nodes=n_gpus if wl.get("inter_intra") else 0, peer_group=pg,
                            nvls=args.nvls if n_gpus > 1 else 0, dtype=wl.get("dtype", "f32"))
    # steps are issued by the library's native lockstep executor (rp_lockstep_run: the same
    # public calls as runner.step(), from C++); --per-call drives them from Python instead
    step_fn = runner.step if args.per_call else (lambda: runner.run_native(1))
    if args.per_call:
        for _ in range(args.warmup):
            runner.step()
    else:
        runner.run_native(args.warmup)
    runner.synchronize()
    runner.ctx.timing_read()                              # drop warm-up launches
    s0 = torch.cuda.ExternalStream(runner.streams[runner.local[0]])   # every batch launches here
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st0 = runner.ctx.stats()
    barrier(pg)
    with ClockSampler(local_rank) as clk:
        runner.synchronize()
        ev0.record(s0)
        if args.per_call:
            for _ in range(args.steps):
                runner.step()
        else:
            runner.run_native(args.steps)
        ev1.record(s0)
        runner.synchronize()
    barrier(pg)
    st1 = runner.ctx.stats()
    ms = max_over_ranks(ev0.elapsed_time(ev1), pg)
    tim = runner.ctx.timing_read()
    launches = st1["kernel_launches"] - st0["kernel_launches"]
    per_rank = gather({"tim": tim, "launches": launches, "clocks": clk.summary(),
                       "hbm": st1["bytes_hbm"] - st0["bytes_hbm"],
                       "nvl": st1["bytes_nvlink"] - st0["bytes_nvlink"],
                       "cross": st1["cross_gpu_groups"] - st0["cross_gpu_groups"]}, pg)
    e2e = run_e2e(runner, args, torch, pg, step_fn)
    runner.close()
    if rank != 0:
        return
    value = world * args.steps / (ms / 1e3)
    peaks, peak_src = measured_peaks()
    hbm_step = sum(r["hbm"] for r in per_rank) / args.steps
    nvl_step = sum(r["nvl"] for r in per_rank) / args.steps
    loc_ms = sum(r["tim"]["local_ms"] for r in per_rank)
    loc_b = sum(r["tim"]["local_bytes_hbm"] for r in per_rank)
    x_ms = sum(r["tim"]["cross_ms"] for r in per_rank)
    x_b = sum(r["tim"]["cross_bytes_nvlink"] for r in per_rank)
    hbm_roof = None
    if loc_ms > 0:
        a = loc_b / (loc_ms / 1e3) / 1e9
        hbm_roof = {"bound": "hbm",
                    "kernel": "preduce_dyn_kernel (fused SGD + P-Reduce, intra-GPU groups, TMA bulk copies, "
                              "warp-specialized, dynamic tiles)",
                    "achieved": round(a, 1), "peak": peaks["hbm_gbs"], "peak_source": peak_src, "unit": "GB/s",
                    "frac": round(a / peaks["hbm_gbs"], 4),
                    # the measured peak is a torch copy (1:1 read:write); this kernel streams 2:1
                    # read:write, which the HBM serves faster, so frac can exceed 1
                    "frac_of_nominal": round(a / HBM_NOMINAL, 4),
                    "traffic": traffic_from_profiles(args.workload, n_gpus),
                    "launches": sum(r["tim"]["local_launches"] for r in per_rank),
                    "kernel_ms_per_launch": round(loc_ms / max(1, sum(r["tim"]["local_launches"] for r in per_rank)), 4),
                    "algorithmic_bytes_per_launch": int(loc_b / max(1, sum(r["tim"]["local_launches"] for r in per_rank)))}
    nvl_roof = None
    if x_ms > 0:
        # the cross-GPU kernel moves NVLink bytes and (fused intra-GPU groups, pre-reduction)
        # HBM bytes; its bound is whichever resource it uses the larger fraction of
        a = x_b / (x_ms / 1e3) / 1e9        # per GPU: its NVLink bytes / its kernel time
        xh = sum(r["tim"]["cross_bytes_hbm"] for r in per_rank)
        ah = xh / (x_ms / 1e3) / 1e9
        nl = sum(r["tim"]["cross_launches"] for r in per_rank)
        kname = "xgpu_kernel (fused SGD + P-Reduce, cross-GPU part)"
        if args.nvls:
            kname = f"nvls_kernel (in-switch P-Reduce, groups on >= {args.nvls} GPUs) + " + kname
        nvl_roof = {"bound": "nvlink", "kernel": kname,
                    "achieved": round(a, 1), "peak": NVLINK_PEAK,
                    "peak_source": "fallback (B200_PROFILING.md: measured peer copy per direction; 900 nominal)",
                    "unit": "GB/s", "frac": round(a / NVLINK_PEAK, 4), "frac_of_nominal": round(a / NVLINK_NOMINAL, 4),
                    "traffic": None, "launches": nl,
                    "kernel_ms_per_launch": round(x_ms / max(1, nl), 4),
                    "algorithmic_nvlink_bytes_per_launch_per_gpu": int(x_b / max(1, nl)),
                    "hbm_achieved": round(ah, 1), "hbm_frac": round(ah / peaks["hbm_gbs"], 4)}
        # the schedule may load GPUs unequally (e.g. SHIFT_K with 2 workers/GPU puts some GPUs
        # in two cross-GPU groups per step): the GPU with the most NVLink bytes sets the pace
        busy = max(per_rank, key=lambda r: r["tim"]["cross_bytes_nvlink"])
        if busy["tim"]["cross_ms"] > 0:
            ab = busy["tim"]["cross_bytes_nvlink"] / (busy["tim"]["cross_ms"] / 1e3) / 1e9
            nvl_roof["busiest_gpu"] = {"achieved": round(ab, 1), "frac": round(ab / NVLINK_PEAK, 4),
                                       "nvlink_bytes": int(busy["tim"]["cross_bytes_nvlink"]),
                                       "share_of_all_nvlink_bytes": round(busy["tim"]["cross_bytes_nvlink"] /
                                                                          max(1, x_b), 4)}
        if ah / peaks["hbm_gbs"] > a / NVLINK_PEAK:      # fused local work dominates: HBM-bound
            nvl_roof.update({"bound": "hbm", "achieved": round(ah, 1), "peak": peaks["hbm_gbs"],
                             "peak_source": peak_src, "frac": round(ah / peaks["hbm_gbs"], 4),
                             "nvlink_achieved": round(a, 1), "nvlink_frac": round(a / NVLINK_PEAK, 4)})
    # the dominant kernel is the one with the larger share of device time
    main_is_nvl = bool(nvl_roof) and x_ms >= loc_ms
    roof = nvl_roof if main_is_nvl else (hbm_roof or nvl_roof)
    if roof is not None:
        roof = dict(roof)
        roof["other_kernel"] = hbm_roof if main_is_nvl else nvl_roof
    clocks = [r["clocks"] for r in per_rank if r["clocks"]]
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
        "dtype": "f32",                         # arithmetic; storage in config.storage
        "data": "synthetic (counter-based xi generator; resident replicas + gradients)",
        "impl": "ours",
        "preduce_gbs": round((hbm_step + nvl_step) * args.steps / (ms / 1e3) / 1e9, 1),
        "config": {"workload": args.workload, "desc": wl["desc"], "world": world, "workers_per_gpu": wpg,
                   "n_params": n, "group_size": k, "schedule": wl["rule"] or "GB+GD (lockstep, ascending requests)",
                   "driver": "per-call API from Python" if args.per_call else "rp_lockstep_run (native executor)",
                   "lr": 0.1, "hbm_bytes_per_step": int(hbm_step), "nvlink_bytes_per_step": int(nvl_step),
                   "cross_gpu_groups_per_step": sum(r["cross"] for r in per_rank) / args.steps,
                   "nvls_min_gpus": args.nvls if n_gpus > 1 else 0,
                   "storage": wl.get("dtype", "f32"),
                   "parallelism": f"{n_gpus} ranks x {wpg} workers, disjoint groups",
                   "l2": ("inputs larger than L2" if hbm_step / n_gpus > L2_BYTES else
                          "working set fits in L2 (no flush): L2-resident number")},
        "roofline": roof,
        "gpu_launches": sum(r["launches"] for r in per_rank),
        "clocks": clocks[0] if len(clocks) == 1 else {
            "sm_mhz": statistics.median(c["sm_mhz"] for c in clocks),
            "sm_max_mhz": max(c["sm_max_mhz"] for c in clocks),
            "reasons": sorted({x for c in clocks for x in c["reasons"]}), "per_rank": clocks} if clocks else None,
        "e2e": e2e,
    }
    if n_gpus == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(wl, n_gpus, budget_s=args.cpu_budget)
    print(json.dumps(out), flush=True)


def run_async(args, wl):
    """configs[4]: one host thread per worker, one shared GG, synthetic compute T_c per step on
    the worker's stream (slowed worker: (1 + s) T_c, reading R13), for a fixed wall-clock window;
    value = worker-steps completed inside the window / window, all ranks."""
    import random
    import torch
    import paper_1909_08029_b200 as rp
    from paper_1909_08029_b200.async_runner import AsyncRunner

    rank, local_rank, n_gpus = init_dist(args)
    torch.cuda.set_device(local_rank)
    pg = setup_dist(n_gpus, local_rank)
    wpg, n = wl["wpg"], wl["n"]
    world = wpg * n_gpus
    k = min(wl["k"], world)
    job = [random.getrandbits(62) + 1]
    if pg is not None:
        import torch.distributed as dist
        dist.broadcast_object_list(job, src=0, group=pg)
    if args.k:
        k = min(args.k, world)
    r = AsyncRunner(world, n, group_size=k, c_thres=4, seed_gd=3, n_gpus=n_gpus, rank=rank, device=local_rank,
                    job_id=job[0], peer_group=pg, grad_mode="resident", flags=rp.RP_FLAG_TIMING, policy=args.gg,
                    nvls=args.nvls if n_gpus > 1 else 0)
    tc = int(args.tc_us * 1000)
    slow = float(args.slow)

    def delay(w):
        return int(tc * (1 + slow)) if w == 0 else tc
    r.run(steps=max(3, args.warmup), delay_ns=delay, delay_mode=args.delay)   # warm-up, then all retired
    r.close()
    r = AsyncRunner(world, n, group_size=k, c_thres=4, seed_gd=3, n_gpus=n_gpus, rank=rank, device=local_rank,
                    job_id=job[0] + 1, peer_group=pg, grad_mode="resident", flags=rp.RP_FLAG_TIMING, policy=args.gg,
                    nvls=args.nvls if n_gpus > 1 else 0)
    barrier(pg)
    with ClockSampler(local_rank) as clk:
        done = r.run(window_s=args.window, delay_ns=delay, delay_mode=args.delay)
    st = r.ctx.stats()
    tim = r.ctx.timing_read()
    per_rank = gather({"done": done, "tim": tim, "st": st, "clocks": clk.summary()}, pg)
    r.close()
    if rank != 0:
        return
    steps = {w: v for d in per_rank for w, v in d["done"].items()}
    total = sum(steps.values())
    x_ms = sum(d["tim"]["cross_ms"] for d in per_rank)
    x_b = sum(d["tim"]["cross_bytes_nvlink"] for d in per_rank)
    out = {
        "metric": "worker-steps/s (P-Reduce GB/s vs NVLink/HBM roofline; worker-steps/sec at 1/2/4/8 B200)",
        "value": round(total / args.window, 1), "unit": "worker-steps/s", "n_gpus": n_gpus,
        "steps": total, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "impl": "ours", "data": "synthetic",
        "config": {"workload": args.workload, "desc": wl["desc"], "world": world, "workers_per_gpu": wpg,
                   "n_params": n, "group_size": k, "c_thres": 4, "slow_factor": slow, "tc_us": args.tc_us,
                   "group_generation": ("random GG + lock vector + pending queue (P:680-745)" +
                                        (" = AD-PSGD" if k == 2 else "")) if args.gg == "random"
                                       else "GB + GD + slowdown filter (P:997-1195)",
                   "gg_pending": sum(d["st"]["gg_pending"] for d in per_rank),
                   "gg_granted": sum(d["st"]["gg_granted"] for d in per_rank),
                   "compute": f"{args.delay} delay per step (T_c; worker 0: (1 + slow) T_c)",
                   "window_s": args.window,
                   "steps_per_worker": [steps[w] for w in sorted(steps)],
                   "gd_calls": per_rank[0]["st"]["gd_calls"],
                   "cross_gpu_groups": sum(d["st"]["cross_gpu_groups"] for d in per_rank),
                   "groups_launched": sum(d["st"]["groups_launched"] for d in per_rank)},
        "roofline": ({"bound": "nvlink", "kernel": "xgpu_kernel (async cross-GPU groups)",
                      "achieved": round(x_b / (x_ms / 1e3) / 1e9, 1), "peak": NVLINK_PEAK, "unit": "GB/s",
                      "frac": round(x_b / (x_ms / 1e3) / 1e9 / NVLINK_PEAK, 4)} if x_ms > 0 else None),
        "gpu_launches": sum(d["st"]["kernel_launches"] for d in per_rank),
        "clocks": next((d["clocks"] for d in per_rank if d["clocks"]), None),
        "e2e": None,
    }
    print(json.dumps(out), flush=True)


def run_nccl_ar(args, wl):
    """Baseline: global All-Reduce (Horovod/NCCL in the paper) of every
    worker's SGD-updated replica: local SGD + pre-sum of the GPU's workers, ncclAllReduce(sum),
    divide by the world size, write back to every local replica (torch ops + NCCL)."""
    import torch
    import torch.distributed as dist

    rank, local_rank, n_gpus = init_dist(args)
    torch.cuda.set_device(local_rank)
    if n_gpus > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        pg = dist.new_group(backend="gloo")
    else:
        pg = None
    wpg, n = wl["wpg"], wl["n"]
    world = wpg * n_gpus
    X = torch.rand((wpg, n), device="cuda") * 2 - 1
    G = torch.rand((wpg, n), device="cuda") * 2 - 1
    lr = 0.1

    stream = torch.cuda.current_stream()
    delay_ns = 0
    if wl["mode"] == "async":       # configs[4]: every step waits for the slowest worker's compute
        import paper_1909_08029_b200 as rp
        tc = int(args.tc_us * 1000)
        delay_ns = int(tc * (1 + float(args.slow))) if rank == 0 else tc

    def step():
        if delay_ns:
            if args.delay == "host":
                # synchronous training: compute of step t+1 starts from the averaged step-t model
                torch.cuda.current_stream().synchronize()
                time.sleep(delay_ns / 1e9)
            else:
                rp.compute_delay(stream.cuda_stream, delay_ns)
        X.sub_(G, alpha=lr)
        s = X.sum(0) if wpg > 1 else X[0].clone()
        if n_gpus > 1:
            dist.all_reduce(s)
        s.div_(world)
        X.copy_(s.expand_as(X))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(pg)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    barrier(pg)
    ms = max_over_ranks(ev0.elapsed_time(ev1), pg)
    if rank == 0:
        bus = 2 * (n_gpus - 1) / n_gpus * 4 * n if n_gpus > 1 else 0
        print(json.dumps({
            "metric": "worker-steps/s (P-Reduce GB/s vs NVLink/HBM roofline; worker-steps/sec at 1/2/4/8 B200)",
            "value": round(world * args.steps / (ms / 1e3), 1), "unit": "worker-steps/s", "n_gpus": n_gpus,
            "slow_factor": float(args.slow) if wl["mode"] == "async" else None,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
            "higher_is_better": True, "scaling": "weak", "dtype": "f32", "impl": "nccl-allreduce-baseline",
            "busbw_gbs": round(bus * args.steps / (ms / 1e3) / 1e9, 1) if bus else None,
            "config": {"workload": args.workload, "world": world, "workers_per_gpu": wpg, "n_params": n}}),
            flush=True)


def run_e2e(runner, args, torch, pg, step_fn):
    """Same metric through the public API with host buffers: per step, h2d of every local worker's
    gradient from pinned host memory, the lockstep step, and a blocking d2h read of the step's
    result (the first 4 averaged parameters of every local worker). Max over ranks."""
    steps = max(1, min(args.steps, args.e2e_steps))
    n = runner.n
    gdt = runner.G.dtype
    host_g = [torch.empty(n, dtype=gdt, pin_memory=True) for _ in runner.local]
    for i, w in enumerate(runner.local):
        host_g[i].copy_(runner.g(w), non_blocking=False)
    host_out = torch.empty((len(runner.local), 4), dtype=runner.X.dtype, pin_memory=True)
    runner.synchronize()
    streams = {w: torch.cuda.ExternalStream(runner.streams[w]) for w in runner.local}
    barrier(pg)
    t0 = time.perf_counter()
    for _ in range(steps):
        for i, w in enumerate(runner.local):
            with torch.cuda.stream(streams[w]):
                runner.g(w).copy_(host_g[i], non_blocking=True)
        step_fn()
        for i, w in enumerate(runner.local):
            with torch.cuda.stream(streams[w]):
                host_out[i].copy_(runner.x(w)[:4], non_blocking=True)
        for w in runner.local:
            streams[w].synchronize()
    dt = max_over_ranks(time.perf_counter() - t0, pg)
    return {"value": round(runner.world * steps / dt, 1) if dt > 0 else None,
            "unit": "worker-steps/s", "steps": steps,
            "h2d_bytes_per_step": host_g[0].element_size() * n * runner.world,
            "d2h_bytes_per_step": 4 * host_out.element_size() * runner.world,
            "timer": "host wall clock around the public-API steps (includes pinned h2d/d2h), max over ranks"}


def traffic_from_profiles(workload, n_gpus):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel, from the
    committed ncu --set full capture of this workload (profiles/traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(f"{workload}@{n_gpus}")
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
    from oracle.update import bf16_round, fused_group_update, fused_group_update_bf16
    from rp_inputs import gen

    world = wl["wpg"] * n_gpus
    X = {w: gen.x0(w, wl["n"], 0, sample) for w in range(world)}
    G = {w: gen.grad(w, 1, wl["n"], 0, sample) for w in range(world)}
    bf = wl.get("dtype") == "bf16"
    if bf:
        X = {w: bf16_round(v) for w, v in X.items()}
        G = {w: bf16_round(v) for w, v in G.items()}
    k = min(wl["k"], world)
    gg = (GroupGenerator(world, k, c_thres=4, seed_gd=3, nodes=n_gpus if wl.get("inter_intra") else 0)
          if wl["mode"] in ("gd", "async") else None)
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
            groups = S.groups_for(wl["rule"], t, n=world, k=k)
            covered = {w for g in groups for w in g}
            groups = groups + [(w,) for w in range(world) if w not in covered]
        for g in groups:
            if bf:
                fused_group_update_bf16(X, {w: G[w] for w in g}, g, lr, wl["wpg"])
            else:
                fused_group_update(X, {w: G[w] for w in g}, g, lr, wl["wpg"])
    return time.perf_counter() - t0


def cpu_baseline(wl, n_gpus, budget_s=12.0):
    """The oracle as it stands, one host core, bounded sample scaled to the full vector."""
    world = wl["wpg"] * n_gpus
    sample = min(wl["n"], 1 << 20)
    dt = oracle_steps(wl, n_gpus, sample, 1)                        # calibrate
    steps = max(1, min(2000, int(budget_s / max(dt, 1e-6))))
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
    ap.add_argument("--impl", choices=["ours", "reference", "nccl"], default="ours",
                    help="ours | reference (CPU oracle) | nccl (global all-reduce baseline)")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=None)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--nvls", type=int, default=0,
                    help="N>1: cross-GPU groups spanning >= this many GPUs reduce inside the NVSwitch (0 = off)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--per-call", action="store_true",
                    help="drive each lockstep step from Python through the per-call API instead of rp_lockstep_run")
    ap.add_argument("--slow", type=float, default=2.0, help="cfg5: extra delay of worker 0 in units of T_c")
    ap.add_argument("--tc-us", type=float, default=2000.0, help="cfg5: synthetic compute time per step")
    ap.add_argument("--window", type=float, default=3.0, help="cfg5: measured wall-clock window (s)")
    ap.add_argument("--gg", choices=["gd", "random"], default="gd",
                    help="cfg5 group generation: GB+GD+filter (§5) or the random GG of §4.1")
    ap.add_argument("--k", type=int, default=0, help="cfg5: group size override (2 + --gg random = AD-PSGD)")
    ap.add_argument("--delay", choices=["host", "device"], default="host",
                    help="cfg5: synthetic compute as a host sleep (P:1395) or a device busy wait")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.workload is None:
        # N = 1: configs[1] exactly. N > 1: the same layout (8 workers per B200, ResNet-50 size,
        # k = 3, GB + GD) weak-scaled with the paper's architecture-aware GD (§5.2 Inter-Intra,
        # GPU = node), which the paper proposes for nodes of 4-8 workers because random
        # division across nodes congests the interconnect; plain GD over 8N
        # workers stays available as --workload cfg2
        args.workload = "cfg2" if args.gpus == 1 else "cfg2ii"
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, wl)
    elif args.impl == "nccl":
        run_nccl_ar(args, wl)
    elif wl["mode"] == "async":
        run_async(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
