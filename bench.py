#!/usr/bin/env python3
"""Benchmark of the fused SGD + P-Reduce hot path (Ripples, arXiv 1909.08029) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference|nccl|nccl-group]
                    [--workload NAME]

One "step" is one lockstep training iteration of every worker (alg1):
group determination (GB + GD or a static rule) + the fused SGD + P-Reduce kernel(s) for all
groups, with parameter and gradient vectors resident in HBM. Prints ONE JSON line (rank 0).
Metric: worker-steps/s (BASELINE.json: "P-Reduce GB/s vs NVLink/HBM roofline; worker-steps/sec
at 1/2/4/8 B200"); P-Reduce GB/s and the roofline fractions ride along.

Default workload: `r50x8`, the SAME 8 workers (ResNet-50-sized, k = 3, GB + GD) spread over the
N GPUs: N = 1 is BASELINE configs[1], N = 8 is configs[2] (strong scaling). At N > 1 the line
also carries `extras`: configs[3] (cfg4, VGG-16 size, 2 workers per GPU, static SHIFT_K) with
its NVLink roofline, the paper's own per-group NCCL P-Reduce (`nccl-group`) and the global
all-reduce on the same problem, and configs[4] (cfg5, one worker slowed 2x) against all-reduce.

--impl reference times the CPU oracle (test infrastructure; the one other place this file runs
oracle/) on a bounded sample of the same workload. --impl nccl / nccl-group are the NCCL
baselines (global all-reduce; the paper's per-group sub-communicator all-reduce).
"""
import argparse
import json
import os
import statistics
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
METRIC = "worker-steps/s (P-Reduce GB/s vs NVLink/HBM roofline; worker-steps/sec at 1/2/4/8 B200)"

# name -> workload. wpg: workers per GPU (weak scaling); world: a fixed total split over the GPUs
WORKLOADS = {
    "r50x8": dict(desc="configs[1] -> configs[2]: the SAME 8 workers (ResNet-50-sized 25.6M fp32, k=3, GB+GD, "
                       "lockstep requests in ascending order) spread over N B200 (8/N workers per GPU): N=1 is "
                       "configs[1], N=8 is configs[2]",
                  world=8, n=N_R50, k=3, mode="gd", rule=None, scaling="strong"),
    "cfg1": dict(desc="configs[0]: 4 workers, 1M fp32, k=2, static SHIFT_K(4,2), 1 GPU; one schedule period "
                      "captured into a CUDA graph and replayed (RP_FLAG_GRAPH: launch-bound size)",
                 wpg=4, n=1 << 20, k=2, mode="static", rule="shift_k", graph=True),
    "cfg2": dict(desc="configs[1] layout weak-scaled: 8 workers per B200, ResNet-50-sized, k=3, GB+GD over all "
                      "8*N workers (N=1: exactly configs[1])",
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
    "cfg3": dict(desc="configs[2] layout: 1 worker per B200 (8 workers on 8 GPUs), ResNet-50-sized, k=3, GB+GD, "
                      "concurrent disjoint groups over NVLink",
                 wpg=1, n=N_R50, k=3, mode="gd", rule=None),
    "cfg4": dict(desc="configs[3]: 2 workers per B200 (16 on 8 GPUs), VGG-16-sized 138M fp32, k=3, static "
                      "SHIFT_K(2N,3)",
                 wpg=2, n=N_VGG, k=3, mode="static", rule="shift_k"),
    "cfg4p4": dict(desc="configs[3] layout with the paper's architecture-aware static rule PAPER4 (fig:scheduler, "
                        "P:883-923; GPU = node, 2 workers per node)",
                   wpg=2, n=N_VGG, k=3, mode="static", rule="paper4"),
    "xall": dict(desc="diagnostic: 1 worker per B200, ResNet-50-sized, ONE group of all N GPUs every step "
                      "(SHIFT_K(N,N)): the cross-GPU kernel's NVLink efficiency without lockstep skew",
                 wpg=1, n=N_R50, k=64, mode="static", rule="shift_k"),
    "xall_vgg": dict(desc="diagnostic: 1 worker per B200, VGG-16-sized, ONE group of all N GPUs every step",
                     wpg=1, n=N_VGG, k=64, mode="static", rule="shift_k"),
    "xall_vgg_m2": dict(desc="diagnostic: 2 workers per B200, VGG-16-sized, ONE group of all 2N workers every step "
                             "(every GPU pre-reduces 2 members: the HBM-heavy side of configs[3])",
                        wpg=2, n=N_VGG, k=64, mode="static", rule="shift_k"),
    "cfg5": dict(desc="configs[4]: 2 workers per B200, VGG-16-sized, k=3, asynchronous GB+GD+filter (C_thres=4), "
                      "worker 0 slowed by --slow x T_c (P:1395)",
                 wpg=2, n=N_VGG, k=3, mode="async", rule=None),
    "cfg5static": dict(desc="configs[4] layout with the static rule SHIFT_K(2N,3) instead of dynamic GG: per-worker "
                            "synthetic compute T_c on the worker's stream (worker 0: (1 + slow) T_c), group-local "
                            "ordering on the device (the paper's 'static' arm, P:1406-1407)",
                       wpg=2, n=N_VGG, k=3, mode="static", rule="shift_k", delayed=True),
}
NVLINK_PEAK = 770.0   # GB/s per direction, measured peer copy (B200_PROFILING.md)
NVLINK_NOMINAL = 900.0
HBM_NOMINAL = 7700.0  # GB/s, B200 HGX HBM3e (B200_PROFILING.md)


def wpg_of(wl, n_gpus):
    """Workers per GPU: fixed per GPU (weak scaling), or a fixed total world split over the GPUs."""
    if "world" in wl:
        if wl["world"] % n_gpus:
            raise SystemExit(f"workload needs a GPU count dividing {wl['world']}")
        return wl["world"] // n_gpus
    return wl["wpg"]


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


def merge_clocks(clocks):
    clocks = [c for c in clocks if c]
    if not clocks:
        return None
    if len(clocks) == 1:
        return clocks[0]
    return {"sm_mhz": statistics.median(c["sm_mhz"] for c in clocks), "sm_max_mhz": max(c["sm_max_mhz"] for c in clocks),
            "reasons": sorted({x for c in clocks for x in c["reasons"]}), "per_rank": clocks}


# ------------------------------------------------------------------------------------------
# process group (one rank per GPU; NCCL for the baselines, gloo for host metadata)
# ------------------------------------------------------------------------------------------

class Dist:
    def __init__(self, args):
        import torch
        self.n = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        if self.n != args.gpus:
            raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={self.n}")
        torch.cuda.set_device(self.local_rank)
        self.pg = None
        if self.n > 1:
            import torch.distributed as dist
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local_rank))
            self.pg = dist.new_group(backend="gloo")

    def max(self, v):
        import torch
        import torch.distributed as dist
        if self.pg is None:
            return v
        t = torch.tensor([float(v)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.pg)
        return float(t.item())

    def gather(self, obj):
        import torch.distributed as dist
        if self.pg is None:
            return [obj]
        out = [None] * dist.get_world_size(self.pg)
        dist.all_gather_object(out, obj, group=self.pg)
        return out

    def barrier(self):
        import torch.distributed as dist
        if self.pg is not None:
            dist.barrier(group=self.pg)


def free_cuda():
    import gc
    import torch
    gc.collect()
    torch.cuda.empty_cache()


# ------------------------------------------------------------------------------------------
# ours: lockstep (rp_lockstep_run)
# ------------------------------------------------------------------------------------------

def cross_roofline(recs_per_rank, ms_total, steps, peaks, peak_src, gpm):
    """NVLink roofline of the cross-GPU kernel from per-launch records of every rank.

    kernel level: algorithmic NVLink bytes / kernel event time (time includes waiting for peers);
    bottleneck:   per step, the GPU with the most NVLink bytes sets the pace: its bytes / its
                  kernel time in that step (the kernel's rate where the rate matters);
    step level:   sum over steps of max_gpu(bytes) / 770 GB/s, divided by the measured step time
                  (fraction of roofline = T_bound / T_measured)."""
    xs = [[r for r in recs if r["cross"]] for recs in recs_per_rank]
    x_ms = sum(r["ms"] for rs in xs for r in rs)
    x_b = sum(r["bytes_nvlink"] for rs in xs for r in rs)
    x_h = sum(r["bytes_hbm"] for rs in xs for r in rs)
    nl = sum(len(rs) for rs in xs)
    if x_ms <= 0 or nl == 0:
        return None
    a = x_b / (x_ms / 1e3) / 1e9
    by_step = {}
    for rank, rs in enumerate(xs):
        for r in rs:
            e = by_step.setdefault(r["batch"], {})
            b, ms = e.get(rank, (0, 0.0))
            e[rank] = (b + r["bytes_nvlink"], ms + r["ms"])
    bott_b = bott_ms = bound_s = 0.0
    for e in by_step.values():
        rank = max(e, key=lambda q: e[q][0])
        bott_b += e[rank][0]
        bott_ms += e[rank][1]
        bound_s += e[rank][0] / (NVLINK_PEAK * 1e9)
    ab = bott_b / (bott_ms / 1e3) / 1e9 if bott_ms > 0 else None
    busy = max(range(len(xs)), key=lambda q: sum(r["bytes_nvlink"] for r in xs[q]))
    bb = sum(r["bytes_nvlink"] for r in xs[busy])
    bms = sum(r["ms"] for r in xs[busy])
    out = {"bound": "nvlink", "kernel": "xgpu_kernel (fused SGD + P-Reduce, cross-GPU part: lane-pipelined "
                                        "reduce-scatter + all-gather, TMA bulk stores over NVLink)",
           "achieved": round(ab if ab else a, 1), "peak": NVLINK_PEAK,
           "peak_source": "B200_PROFILING.md measured peer copy per direction (900 nominal)",
           "unit": "GB/s", "frac": round((ab if ab else a) / NVLINK_PEAK, 4),
           "frac_of_nominal": round((ab if ab else a) / NVLINK_NOMINAL, 4),
           "achieved_definition": "per step, the GPU with the most NVLink bytes: its algorithmic NVLink bytes / "
                                  "its cross-kernel event time, summed over steps",
           "kernel_level": {"achieved": round(a, 1), "frac": round(a / NVLINK_PEAK, 4),
                            "definition": "all ranks' algorithmic NVLink bytes / all ranks' cross-kernel time "
                                          "(includes waiting for peers still in their previous step)"},
           "busiest_gpu": {"rank": busy, "achieved": round(bb / (bms / 1e3) / 1e9, 1) if bms > 0 else None,
                           "frac": round(bb / (bms / 1e3) / 1e9 / NVLINK_PEAK, 4) if bms > 0 else None,
                           "nvlink_bytes": int(bb)},
           "step_level": {"t_bound_ms_per_step": round(bound_s * 1e3 / steps, 4),
                          "ms_per_step": round(ms_total / steps, 4),
                          "frac": round(bound_s * 1e3 / ms_total, 4) if ms_total > 0 else None},
           "launches": nl, "kernel_ms_per_launch": round(x_ms / nl, 4),
           "algorithmic_nvlink_bytes_per_launch_per_gpu": int(x_b / nl),
           "hbm_achieved": round(x_h / (x_ms / 1e3) / 1e9, 1),
           "traffic": None}
    if gpm and all(g and g.get("tx_bytes") is not None for g in gpm):
        alg = [sum(r["bytes_nvlink"] for r in rs) for rs in xs]
        tx = [g["tx_bytes"] for g in gpm]
        out["traffic"] = {"source": gpm[0]["source"], "measured_tx_bytes_per_step": [int(v / steps) for v in tx],
                          "measured_rx_bytes_per_step": [int((g.get("rx_bytes") or 0) / steps) for g in gpm],
                          "algorithmic_bytes_per_step": [int(v / steps) for v in alg],
                          "measured_over_algorithmic": round(sum(tx) / max(1, sum(alg)), 4)}
    elif gpm:
        out["traffic"] = {"unavailable": sorted({(g or {}).get("error") or "no sample" for g in gpm}),
                          "note": "nvmlDeviceGetFieldValues NVLink counters: NOT_SUPPORTED on these boxes; "
                                  "ncu cannot wrap a multi-rank run (profiles/r02_nvlink_counters.md)"}
    return out


def hbm_roofline(recs_per_rank, peaks, peak_src, workload, n_gpus):
    ls = [r for recs in recs_per_rank for r in recs if not r["cross"]]
    ms = sum(r["ms"] for r in ls)
    if ms <= 0:
        return None
    b = sum(r["bytes_hbm"] for r in ls)
    a = b / (ms / 1e3) / 1e9
    return {"bound": "hbm",
            "kernel": "preduce_dyn_kernel (fused SGD + P-Reduce, intra-GPU groups, TMA bulk copies, "
                      "warp-specialized, dynamic tiles)",
            "achieved": round(a, 1), "peak": peaks["hbm_gbs"], "peak_source": peak_src, "unit": "GB/s",
            "frac": round(a / peaks["hbm_gbs"], 4),
            # the measured peak is a torch copy (1:1 read:write); this kernel streams 2:1 read:write,
            # which the HBM serves faster, so frac can exceed 1
            "frac_of_nominal": round(a / HBM_NOMINAL, 4),
            "traffic": traffic_from_profiles(workload, n_gpus),
            "launches": len(ls), "kernel_ms_per_launch": round(ms / len(ls), 4),
            "algorithmic_bytes_per_launch": int(b / len(ls))}


def run_ours(args, wl, name, D, steps=None, warmup=None, e2e=True, delay_us=None):
    """Lockstep workload through rp_lockstep_run; returns the JSON dict on rank 0, else None."""
    import torch
    import paper_1909_08029_b200 as rp
    from paper_1909_08029_b200.nvlink_counters import GpmNvlink
    from paper_1909_08029_b200.runner import LockstepRunner

    steps = steps or args.steps
    warmup = warmup or args.warmup
    n_gpus, rank = D.n, D.rank
    wpg, n = wpg_of(wl, n_gpus), wl["n"]
    world = wpg * n_gpus
    k = min(wl["k"], world)              # e.g. one group of all GPUs for xall
    flags = rp.RP_FLAG_TIMING | (rp.RP_FLAG_INTER_INTRA if wl.get("inter_intra") else 0)
    if wl.get("graph") and n_gpus == 1 and not args.per_call:
        flags |= rp.RP_FLAG_GRAPH
    nodes = n_gpus if (wl.get("inter_intra") or wl["rule"] == "paper4") else 0
    runner = LockstepRunner(world, n, mode=wl["mode"], rule=wl["rule"], group_size=k, n_gpus=n_gpus,
                            rank=rank, device=D.local_rank, grad_mode="resident", flags=flags, nodes=nodes,
                            peer_group=D.pg, nvls=args.nvls if n_gpus > 1 else 0, dtype=wl.get("dtype", "f32"))
    if delay_us is not None:         # synthetic compute per step on each worker's stream (reading R13)
        for w in runner.local:
            runner.ctx.set_compute_delay(w, int(delay_us(w) * 1e3))
    step_fn = runner.step if args.per_call else (lambda: runner.run_native(1))
    if args.per_call:
        for _ in range(warmup):
            runner.step()
    else:
        runner.run_native(warmup)
    runner.synchronize()
    runner.ctx.timing_records()                               # drop warm-up launches
    s0 = torch.cuda.ExternalStream(runner.streams[runner.local[0]])   # every batch launches here
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st0 = runner.ctx.stats()
    gpm = GpmNvlink(D.local_rank) if n_gpus > 1 else None
    D.barrier()
    with ClockSampler(D.local_rank) as clk:
        runner.synchronize()
        if gpm:
            gpm.start()
        ev0.record(s0)
        h0 = time.perf_counter()
        if args.per_call:
            for _ in range(steps):
                runner.step()
        else:
            runner.run_native(steps)
        host_ms = (time.perf_counter() - h0) * 1e3      # host enqueue time of the K steps (no sync)
        ev1.record(s0)
        runner.synchronize()
        g = gpm.stop() if gpm else None
    D.barrier()
    if gpm:
        gpm.close()
    st1 = runner.ctx.stats()
    ms = D.max(ev0.elapsed_time(ev1))
    recs = runner.ctx.timing_records()
    launches = st1["kernel_launches"] - st0["kernel_launches"]
    per_rank = D.gather({"recs": recs, "launches": launches, "clocks": clk.summary(), "gpm": g, "host_ms": host_ms,
                         "hbm": st1["bytes_hbm"] - st0["bytes_hbm"], "nvl": st1["bytes_nvlink"] - st0["bytes_nvlink"],
                         "cross": st1["cross_gpu_groups"] - st0["cross_gpu_groups"]})
    if os.environ.get("RP_BENCH_DUMP_RECS") and rank == 0:   # debugging: every rank's per-launch records
        with open(os.environ["RP_BENCH_DUMP_RECS"], "w") as f:
            json.dump([r["recs"] for r in per_rank], f)
    e2e_line = run_e2e(runner, args, D, step_fn) if e2e else None
    runner.close()
    del runner
    free_cuda()
    if rank != 0:
        return None
    value = world * steps / (ms / 1e3)
    peaks, peak_src = measured_peaks()
    hbm_step = sum(r["hbm"] for r in per_rank) / steps
    nvl_step = sum(r["nvl"] for r in per_rank) / steps
    recs_all = [r["recs"] for r in per_rank]
    hroof = hbm_roofline(recs_all, peaks, peak_src, name, n_gpus)
    xroof = cross_roofline(recs_all, ms, steps, peaks, peak_src, [r["gpm"] for r in per_rank] if n_gpus > 1 else None)
    if xroof and args.nvls:
        xroof["kernel"] = f"nvls_kernel (in-switch P-Reduce, groups on >= {args.nvls} GPUs) + " + xroof["kernel"]
    # the dominant kernel is the one with the larger share of device time
    x_ms = sum(r["ms"] for rs in recs_all for r in rs if r["cross"])
    l_ms = sum(r["ms"] for rs in recs_all for r in rs if not r["cross"])
    main_is_x = bool(xroof) and x_ms >= l_ms
    roof = xroof if main_is_x else (hroof or xroof)
    if roof is not None:
        roof = dict(roof)
        roof["other_kernel"] = hroof if main_is_x else xroof
    elif hbm_step > 0:        # CUDA-graph replay (RP_FLAG_GRAPH): no per-launch events, whole step
        a = hbm_step / (ms / steps / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": "whole lockstep step (CUDA graph replay of the fused SGD + P-Reduce "
                                          "launches; per-launch events are not captured)",
                "achieved": round(a, 1), "peak": peaks["hbm_gbs"], "peak_source": peak_src, "unit": "GB/s",
                "frac": round(a / peaks["hbm_gbs"], 4), "frac_of_nominal": round(a / HBM_NOMINAL, 4),
                "traffic": traffic_from_profiles(name, n_gpus), "algorithmic_bytes_per_step": int(hbm_step)}
    return {
        "metric": METRIC, "value": round(value, 1), "unit": "worker-steps/s", "n_gpus": n_gpus,
        "steps": steps, "warmup": warmup, "ms_per_step": round(ms / steps, 4), "higher_is_better": True,
        "scaling": wl.get("scaling", "weak"), "vs_baseline": None,
        "dtype": "f32",                         # arithmetic; storage in config.storage
        "data": "synthetic (counter-based xi generator; resident replicas + gradients)",
        "impl": "ours",
        "preduce_gbs": round((hbm_step + nvl_step) * steps / (ms / 1e3) / 1e9, 1),
        "config": {"workload": name, "desc": wl["desc"], "world": world, "workers_per_gpu": wpg,
                   "n_params": n, "group_size": k, "schedule": wl["rule"] or "GB+GD (lockstep, ascending requests)",
                   "driver": "per-call API from Python" if args.per_call else "rp_lockstep_run (native executor)",
                   "lr": 0.1, "hbm_bytes_per_step": int(hbm_step), "nvlink_bytes_per_step": int(nvl_step),
                   "cross_gpu_groups_per_step": sum(r["cross"] for r in per_rank) / steps,
                   "nvls_min_gpus": args.nvls if n_gpus > 1 else 0, "storage": wl.get("dtype", "f32"),
                   "parallelism": f"{n_gpus} ranks x {wpg} workers, disjoint groups",
                   "compute_delay_us": None if delay_us is None else {"T_c": args.tc_us, "slow": args.slow},
                   "l2": ("inputs larger than L2" if hbm_step / n_gpus > L2_BYTES else
                          "working set fits in L2 (no flush): L2-resident number")},
        "roofline": roof,
        "gpu_launches": sum(r["launches"] for r in per_rank),
        "clocks": merge_clocks([r["clocks"] for r in per_rank]),
        "host_enqueue_ms": [round(r["host_ms"], 2) for r in per_rank],   # per rank, K steps, no sync
        "e2e": e2e_line,
    }


def run_e2e(runner, args, D, step_fn):
    """Same metric through the public API with host buffers: per step, h2d of every local worker's
    gradient from pinned host memory, the lockstep step, and a blocking d2h copy of every local
    worker's averaged replica (the model the user gets back). Host wall clock, max over ranks."""
    import torch
    steps = max(1, min(args.steps, args.e2e_steps))
    n = runner.n
    host_g = [torch.empty(n, dtype=runner.G.dtype, pin_memory=True) for _ in runner.local]
    host_x = [torch.empty(n, dtype=runner.X.dtype, pin_memory=True) for _ in runner.local]
    for i, w in enumerate(runner.local):
        host_g[i].copy_(runner.g(w), non_blocking=False)
    runner.synchronize()
    streams = {w: torch.cuda.ExternalStream(runner.streams[w]) for w in runner.local}
    D.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        for i, w in enumerate(runner.local):
            with torch.cuda.stream(streams[w]):
                runner.g(w).copy_(host_g[i], non_blocking=True)
        step_fn()
        for i, w in enumerate(runner.local):
            with torch.cuda.stream(streams[w]):
                host_x[i].copy_(runner.x(w), non_blocking=True)
        for w in runner.local:
            streams[w].synchronize()
    dt = D.max(time.perf_counter() - t0)
    return {"value": round(runner.world * steps / dt, 1) if dt > 0 else None,
            "unit": "worker-steps/s", "steps": steps,
            "h2d_bytes_per_step": host_g[0].element_size() * n * runner.world,
            "d2h_bytes_per_step": host_x[0].element_size() * n * runner.world,
            "copies": "h2d every worker's gradient, d2h every worker's averaged replica, pinned host memory",
            "timer": "host wall clock around the public-API steps, max over ranks"}


# ------------------------------------------------------------------------------------------
# ours: asynchronous (configs[4])
# ------------------------------------------------------------------------------------------

def run_async(args, wl, name, D, slow=None):
    """configs[4]: one host thread per worker, one shared GG, synthetic compute T_c per step
    (slowed worker: (1 + s) T_c, reading R13), for a fixed wall-clock window; value = worker-steps
    completed inside the window / window, all ranks."""
    import random
    import paper_1909_08029_b200 as rp
    from paper_1909_08029_b200.async_runner import AsyncRunner

    n_gpus, rank = D.n, D.rank
    wpg, n = wpg_of(wl, n_gpus), wl["n"]
    world = wpg * n_gpus
    k = min(args.k or wl["k"], world)
    slow = float(args.slow if slow is None else slow)
    job = D.gather(random.getrandbits(62) + 1)[0]
    tc = int(args.tc_us * 1000)

    def delay(w):
        return int(tc * (1 + slow)) if w == 0 else tc

    def make(j):
        return AsyncRunner(world, n, group_size=k, c_thres=4, seed_gd=3, n_gpus=n_gpus, rank=rank,
                           device=D.local_rank, job_id=j, peer_group=D.pg, grad_mode="resident",
                           flags=rp.RP_FLAG_TIMING, policy=args.gg, nvls=args.nvls if n_gpus > 1 else 0)
    r = make(job)
    r.run(steps=max(3, args.warmup), delay_ns=delay, delay_mode=args.delay)   # warm-up, then all retired
    r.close()
    r = make(job + 1)
    D.barrier()
    with ClockSampler(D.local_rank) as clk:
        done = r.run(window_s=args.window, delay_ns=delay, delay_mode=args.delay)
    st = r.ctx.stats()
    recs = r.ctx.timing_records()
    per_rank = D.gather({"done": done, "recs": recs, "st": st, "clocks": clk.summary()})
    r.close()
    del r
    free_cuda()
    if rank != 0:
        return None
    steps = {w: v for d in per_rank for w, v in d["done"].items()}
    total = sum(steps.values())
    xs = [r for d in per_rank for r in d["recs"] if r["cross"]]
    x_ms, x_b = sum(r["ms"] for r in xs), sum(r["bytes_nvlink"] for r in xs)
    return {
        "metric": METRIC, "value": round(total / args.window, 1), "unit": "worker-steps/s", "n_gpus": n_gpus,
        "steps": total, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "impl": "ours", "data": "synthetic",
        "config": {"workload": name, "desc": wl["desc"], "world": world, "workers_per_gpu": wpg,
                   "n_params": n, "group_size": k, "c_thres": 4, "slow_factor": slow, "tc_us": args.tc_us,
                   "group_generation": ("random GG + lock vector + pending queue (P:680-745)" +
                                        (" = AD-PSGD" if k == 2 else "")) if args.gg == "random"
                                       else "GB + GD + slowdown filter (P:997-1195)",
                   "gg_pending": sum(d["st"]["gg_pending"] for d in per_rank),
                   "gg_granted": sum(d["st"]["gg_granted"] for d in per_rank),
                   "compute": f"{args.delay} delay per step (T_c; worker 0: (1 + slow) T_c)",
                   "window_s": args.window, "steps_per_worker": [steps[w] for w in sorted(steps)],
                   "gd_calls": per_rank[0]["st"]["gd_calls"],
                   "cross_gpu_groups": sum(d["st"]["cross_gpu_groups"] for d in per_rank),
                   "groups_launched": sum(d["st"]["groups_launched"] for d in per_rank)},
        "roofline": ({"bound": "nvlink", "kernel": "xgpu_kernel (async cross-GPU groups)",
                      "achieved": round(x_b / (x_ms / 1e3) / 1e9, 1), "peak": NVLINK_PEAK, "unit": "GB/s",
                      "frac": round(x_b / (x_ms / 1e3) / 1e9 / NVLINK_PEAK, 4)} if x_ms > 0 else None),
        "gpu_launches": sum(d["st"]["kernel_launches"] for d in per_rank),
        "clocks": merge_clocks([d["clocks"] for d in per_rank]),
        "e2e": None,
    }


# ------------------------------------------------------------------------------------------
# NCCL baselines
# ------------------------------------------------------------------------------------------

class BaselineState:
    """Replicas / gradients of this rank's workers + the seeded schedule (host-only librp context:
    the same static rule or the same replicated GG as ours, so both arms run the same groups)."""

    def __init__(self, wl, D, delay_ns=0, alloc=True):
        import torch
        from paper_1909_08029_b200 import rp
        self.rp, self.D = rp, D
        self.wpg, self.n = wpg_of(wl, D.n), wl["n"]
        self.world = self.wpg * D.n
        self.k = min(wl["k"], self.world)
        self.wl = wl
        self.t = 0
        nodes = D.n if wl["rule"] == "paper4" else 0
        self.host = rp.Context(self.world, self.n, n_gpus=0, group_size=self.k, c_thres=4, nodes=nodes, seed_gd=3)
        if not alloc:
            return
        ld = (self.n + 63) // 64 * 64
        self.X = torch.empty((self.wpg, ld), device="cuda")
        self.G = torch.empty((self.wpg, ld), device="cuda")
        self.S = torch.empty(ld, device="cuda")          # pre-sum / NCCL buffer
        s = torch.cuda.current_stream().cuda_stream
        self.local = list(range(D.rank * self.wpg, (D.rank + 1) * self.wpg))
        for i, w in enumerate(self.local):
            rp.fill_xi(self.X[i], self.n, 1, w, 0, 0, s)
            rp.fill_xi(self.G[i], self.n, 2, w, 1, 0, s)
        self.delay_ns = delay_ns

    def x(self, w):
        return self.X[self.local.index(w), :self.n]

    def g(self, w):
        return self.G[self.local.index(w), :self.n]

    def groups(self):
        """All groups of the next step (every rank computes the same list), ascending."""
        from paper_1909_08029_b200.runner import RULES
        self.t += 1
        if self.wl["mode"] == "static":
            go, _ = self.host.schedule_static(RULES[self.wl["rule"]], self.t)
            gs = {}
            for w, gi in enumerate(go):
                gs.setdefault(gi if gi >= 0 else -1 - w, []).append(w)
            out = [tuple(v) for v in gs.values()]
        else:
            out = []
            seen = set()
            for g in self.host.group_generate_many(list(range(self.world))):
                if g.seq not in seen:
                    seen.add(g.seq)
                    out.append(tuple(g.member_list()))
            for q in sorted(seen):
                self.host.gg_release(q)
        return sorted(out)

    def close(self):
        self.host.close()


def _timed(D, step, steps, warmup):
    import torch
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    D.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(D.local_rank) as clk:
        ev0.record()
        for _ in range(steps):
            step()
        ev1.record()
        torch.cuda.synchronize()
    D.barrier()
    return D.max(ev0.elapsed_time(ev1)), clk.summary()


def run_nccl_ar(args, wl, name, D, steps=None, warmup=None, delay_us=None):
    """Global All-Reduce baseline (Horovod/NCCL in the paper): per step one
    fused SGD + pre-sum kernel over the GPU's workers (rp_bench_presum), in-place ncclAllReduce
    (sum) of the partial, one kernel writing sum / world to every local replica."""
    import torch
    import torch.distributed as dist
    steps, warmup = steps or args.steps, warmup or args.warmup
    B = BaselineState(wl, D)
    s = torch.cuda.current_stream().cuda_stream
    xs = [B.x(w) for w in B.local]
    gs = [B.g(w) for w in B.local]
    dly = [int(delay_us(w) * 1e3) for w in B.local] if delay_us else None

    def step():
        if dly:
            B.rp.compute_delay(s, max(dly))          # the GPU's slowest worker gates its partial
        B.rp.rp_bench_presum(xs, gs, B.n, 0.1, B.S, s)
        if D.n > 1:
            dist.all_reduce(B.S[:B.n])
        B.rp.rp_bench_scatter_mean(B.S, B.n, float(B.world), xs, s)
    ms, clk = _timed(D, step, steps, warmup)
    B.close()
    del B
    free_cuda()
    if D.rank != 0:
        return None
    bus = 2 * (D.n - 1) / D.n * 4 * wl["n"] if D.n > 1 else 0
    return {"metric": METRIC, "value": round(wpg_of(wl, D.n) * D.n * steps / (ms / 1e3), 1), "unit": "worker-steps/s",
            "n_gpus": D.n, "steps": steps, "warmup": warmup, "ms_per_step": round(ms / steps, 4),
            "higher_is_better": True, "dtype": "f32", "impl": "nccl-allreduce-baseline",
            "busbw_gbs": round(bus * steps / (ms / 1e3) / 1e9, 1) if bus else None, "clocks": clk,
            "config": {"workload": name, "workers_per_gpu": wpg_of(wl, D.n), "n_params": wl["n"],
                       "per_step": "rp_bench_presum (SGD + local pre-sum) -> ncclAllReduce(sum) in place -> "
                                   "rp_bench_scatter_mean (sum / world into every replica)",
                       "compute_delay_us": None if delay_us is None else {"T_c": args.tc_us, "slow": args.slow}}}


def run_nccl_group(args, wl, name, D, steps=None, warmup=None):
    """The paper's own P-Reduce (§6): every group is an NCCL all-reduce on a
    communicator of the group's GPUs (created with ncclCommSplit through torch.distributed.new_group,
    all ranks in the same order; an LRU cache of at most 64 communicators), on the same
    schedule as ours. Per GPU and group: rp_bench_presum of the local members, ncclAllReduce(sum)
    across the group's GPUs (skipped for intra-GPU groups), rp_bench_scatter_mean (sum / |G|)."""
    import collections
    import torch
    import torch.distributed as dist
    steps, warmup = steps or args.steps, warmup or args.warmup
    # the schedule of the whole run (a second host-only GG with the same seed): the GPU subsets
    # of its cross-GPU groups, in order of first use. The paper keeps <= 64 communicators
    # cached, so the warm state is every subset the run needs, up to 64; they are created
    # (ncclCommSplit) and connected (one small all-reduce each) before timing. A run needing
    # more than 64 subsets evicts inside the timed region, as the paper's cache would.
    P = BaselineState(wl, D, alloc=False)
    order = []
    for _ in range(warmup + steps):
        for g in P.groups():
            gpus = tuple(sorted({w // P.wpg for w in g}))
            if len(gpus) > 1 and gpus not in order:
                order.append(gpus)
    P.close()
    B = BaselineState(wl, D)
    s = torch.cuda.current_stream().cuda_stream
    cache = collections.OrderedDict()
    stats = {"created": 0, "evicted": 0, "subsets_in_run": len(order)}
    probe = torch.zeros(1024, device="cuda")

    def comm(gpus):
        if gpus in cache:
            cache.move_to_end(gpus)
            return cache[gpus]
        if len(cache) >= 64:
            old, pg = cache.popitem(last=False)
            dist.destroy_process_group(pg)
            stats["evicted"] += 1
        cache[gpus] = dist.new_group(ranks=list(gpus), backend="nccl")   # collective: all ranks, same order
        stats["created"] += 1
        return cache[gpus]

    for gpus in order[:64]:                  # warm cache: create + connect
        pg = comm(gpus)
        if D.rank in gpus:
            dist.all_reduce(probe, group=pg)
    torch.cuda.synchronize()
    stats["created_before_timing"] = stats["created"]

    def step():
        for g in B.groups():
            gpus = tuple(sorted({w // B.wpg for w in g}))
            pg = comm(gpus) if len(gpus) > 1 else None
            if D.rank not in gpus:
                continue
            mine = [w for w in g if w // B.wpg == D.rank]
            buf = B.S                   # groups run one after another in stream order
            B.rp.rp_bench_presum([B.x(w) for w in mine], [B.g(w) for w in mine], B.n, 0.1, buf, s)
            if pg is not None:
                dist.all_reduce(buf[:B.n], group=pg)
            B.rp.rp_bench_scatter_mean(buf, B.n, float(len(g)), [B.x(w) for w in mine], s)
    ms, clk = _timed(D, step, steps, warmup)
    B.close()
    for pg in cache.values():
        dist.destroy_process_group(pg)
    del B
    free_cuda()
    if D.rank != 0:
        return None
    return {"metric": METRIC, "value": round(wpg_of(wl, D.n) * D.n * steps / (ms / 1e3), 1), "unit": "worker-steps/s",
            "n_gpus": D.n, "steps": steps, "warmup": warmup, "ms_per_step": round(ms / steps, 4),
            "higher_is_better": True, "dtype": "f32", "impl": "nccl-group-baseline", "clocks": clk,
            "config": {"workload": name, "workers_per_gpu": wpg_of(wl, D.n), "n_params": wl["n"],
                       "communicators": {"cache_bound": 64, **stats},
                       "per_group": "rp_bench_presum -> ncclAllReduce(sum) on the group's communicator "
                                    "(ncclCommSplit via torch.distributed.new_group) -> rp_bench_scatter_mean"}}


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

def oracle_steps(wl, n_gpus, lo, hi, steps):
    """Time `steps` lockstep steps of the oracle on elements [lo, hi) of every replica, with
    resident gradients like the GPU leg. Returns seconds."""
    import numpy as np
    from oracle import schedule as S
    from oracle.gg import GroupGenerator
    from oracle.update import bf16_round, fused_group_update, fused_group_update_bf16
    from rp_inputs import gen

    wpg = wpg_of(wl, n_gpus)
    world = wpg * n_gpus
    X = {w: gen.x0(w, wl["n"], lo, hi) for w in range(world)}
    G = {w: gen.grad(w, 1, wl["n"], lo, hi) for w in range(world)}
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
            groups = S.groups_for(wl["rule"], t, n=world, k=k, nodes=n_gpus, m=wpg)
            covered = {w for g in groups for w in g}
            groups = groups + [(w,) for w in range(world) if w not in covered]
        for g in groups:
            if bf:
                fused_group_update_bf16(X, {w: G[w] for w in g}, g, lr, wpg)
            else:
                fused_group_update(X, {w: G[w] for w in g}, g, lr, wpg)
    return time.perf_counter() - t0


def _oracle_worker(args):
    wl, n_gpus, lo, hi, steps = args
    return oracle_steps(wl, n_gpus, lo, hi, steps)


def cpu_baseline(wl, n_gpus, budget_s=12.0, all_cores=True):
    """The oracle as it stands on a bounded sample (elements [0, sample) of every replica), one
    host core; optionally also split over every host core (elementwise, so the
    element range splits exactly). Worker-steps/s scaled from the sample to the full vector."""
    world = wpg_of(wl, n_gpus) * n_gpus
    sample = min(wl["n"], 1 << 20)
    dt = oracle_steps(wl, n_gpus, 0, sample, 1)                        # calibrate
    steps = max(1, min(2000, int(budget_s / max(dt, 1e-6))))
    dt = oracle_steps(wl, n_gpus, 0, sample, steps)
    value = world * steps / dt * (sample / wl["n"])
    out = {"value": round(value, 3), "unit": "worker-steps/s", "cores": 1, "kind": "oracle",
           "sample": f"{world} workers x elements [0,{sample}) of {wl['n']}, {steps} steps in {dt:.1f} s; "
                     f"value scaled by {sample}/{wl['n']}",
           "cpu": cpu_model()}
    if all_cores:
        import multiprocessing as mp
        P = max(1, os.cpu_count() or 1)
        per = (wl["n"] + P - 1) // P
        big = min(wl["n"], per * P)
        # every core takes a 1M-element slice of its own stretch of the vector (bounded sample)
        chunks = [(wl, n_gpus, i * per, min(i * per + min(per, 1 << 20), wl["n"]), max(1, steps // 4))
                  for i in range(P) if i * per < big]
        ctx = mp.get_context("fork")
        with ctx.Pool(len(chunks)) as pool:
            t0 = time.perf_counter()
            pool.map(_oracle_worker, chunks)
            wall = time.perf_counter() - t0
        elems = sum(c[3] - c[2] for c in chunks)
        out["all_cores"] = {"value": round(world * chunks[0][4] / wall * (elems / wl["n"]), 3),
                            "unit": "worker-steps/s", "cores": len(chunks),
                            "sample": f"{len(chunks)} processes x <= 1M-element slices ({elems} elements), "
                                      f"{chunks[0][4]} steps, wall {wall:.1f} s; scaled by {elems}/{wl['n']}"}
    return out


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip() + f" ({os.cpu_count()} logical cores on host)"
    except OSError:
        pass
    return None


def run_reference(args, wl, name):
    """The reference arm of this tier: the CPU oracle as it stands, one host core, each step a
    bounded sample (262,144 elements of every replica). `ms_per_step` is what was measured on the
    sample; `value` (and ms_per_step_scaled) extrapolate it to the full vector, labelled as such."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    n_gpus = args.gpus
    world = wpg_of(wl, n_gpus) * n_gpus
    sample = min(wl["n"], 1 << 18)
    for _ in range(args.warmup):
        oracle_steps(wl, n_gpus, 0, sample, 1)
    dts = [oracle_steps(wl, n_gpus, 0, sample, 1) for _ in range(args.steps)]
    dt = sum(dts)
    scale = wl["n"] / sample
    value = world * args.steps / (dt * scale)
    cb = {"value": round(value, 3), "unit": "worker-steps/s", "cores": 1, "kind": "oracle",
          "sample": f"each step: {world} workers x elements [0,{sample}) of {wl['n']}; measured "
                    f"{dt / args.steps * 1e3:.3f} ms per sample step; value scaled by {sample}/{wl['n']}",
          "cpu": cpu_model()}
    return {"metric": METRIC, "value": cb["value"], "unit": "worker-steps/s", "n_gpus": n_gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3),
            "ms_per_step_measured_on": f"{sample}-element sample of every replica",
            "ms_per_step_scaled": round(dt / args.steps * 1e3 * scale, 3),
            "value_is_scaled": True,
            "higher_is_better": True, "scaling": wl.get("scaling", "weak"), "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": name, "desc": wl["desc"], "world": world, "n_params": wl["n"],
                       "group_size": wl["k"]},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "worker-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ------------------------------------------------------------------------------------------

def summary(line, keys=("value", "ms_per_step")):
    if line is None:
        return None
    out = {k: line.get(k) for k in keys}
    r = line.get("roofline")
    if r:
        out["roofline"] = {k: r.get(k) for k in ("bound", "achieved", "frac", "step_level", "kernel_level",
                                                 "busiest_gpu", "traffic") if k in r}
    return out


def extras(args, D):
    """N > 1: configs[3] with its NVLink roofline, the NCCL baselines on the default problem,
    configs[4] slowed run vs all-reduce. Each arm is a short run of its own."""
    ex = {}
    st, wu = min(args.steps, args.extra_steps), 3
    if D.n >= 2:
        ours = run_ours(args, WORKLOADS["cfg4"], "cfg4", D, steps=st, warmup=wu, e2e=False)
        ar = run_nccl_ar(args, WORKLOADS["cfg4"], "cfg4", D, steps=st, warmup=wu)
        if D.rank == 0:
            ex["cfg4"] = {"desc": WORKLOADS["cfg4"]["desc"], "ours": summary(ours), "allreduce": summary(ar),
                          "ours_over_allreduce": round(ours["value"] / ar["value"], 3)}
        grp = run_nccl_group(args, WORKLOADS["r50x8"], "r50x8", D, steps=st, warmup=wu)
        ar8 = run_nccl_ar(args, WORKLOADS["r50x8"], "r50x8", D, steps=st, warmup=wu)
        if D.rank == 0:
            ex["r50x8_baselines"] = {"nccl_group": summary(grp), "allreduce": summary(ar8),
                                     "nccl_group_communicators": grp["config"]["communicators"]}
        tc = args.tc_us
        slow = 2.0

        def dly(w):
            return tc * (1 + slow) if w == 0 else tc
        a5 = run_async(args, WORKLOADS["cfg5"], "cfg5", D, slow=slow)
        ar5 = run_nccl_ar(args, WORKLOADS["cfg5"], "cfg5", D, steps=max(10, st // 2), warmup=wu,
                          delay_us=dly)
        if D.rank == 0:
            ex["cfg5_slowed_2x"] = {"desc": WORKLOADS["cfg5"]["desc"], "ours_gd_async": summary(a5),
                                    "allreduce": summary(ar5),
                                    "ours_over_allreduce": round(a5["value"] / ar5["value"], 3),
                                    "compute": f"T_c = {tc} us ({args.delay} delay in ours; device delay in "
                                               "all-reduce), worker 0: 3 T_c"}
    return ex


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference", "nccl", "nccl-group"], default="ours",
                    help="ours | reference (CPU oracle) | nccl (global all-reduce) | nccl-group (the paper's "
                         "per-group NCCL all-reduce, P:1231-1239)")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="r50x8")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--nvls", type=int, default=0,
                    help="N>1: cross-GPU groups spanning >= this many GPUs reduce inside the NVSwitch (0 = off)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="N>1: skip the cfg4 / NCCL-group / cfg5 extras")
    ap.add_argument("--extra-steps", type=int, default=30)
    ap.add_argument("--no-e2e", action="store_true",
                    help="diagnostics only: skip the e2e measurement (the line then has no e2e number)")
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
    ap.add_argument("--size", type=int, default=0,
                    help="diagnostics only: override the workload's parameter count (the line names it)")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    wl = WORKLOADS[args.workload]
    if args.size > 0:
        wl = dict(wl, n=args.size, desc=wl["desc"] + f" [diagnostic size override: n = {args.size}]")
    if args.impl == "reference":
        line = run_reference(args, wl, args.workload)
        if line:
            print(json.dumps(line), flush=True)
        return
    D = Dist(args)
    if args.impl == "nccl":
        dl = None
        if wl.get("delayed") or wl["mode"] == "async":
            def dl(w):
                return args.tc_us * (1 + args.slow) if w == 0 else args.tc_us
        line = run_nccl_ar(args, wl, args.workload, D, delay_us=dl)
    elif args.impl == "nccl-group":
        line = run_nccl_group(args, wl, args.workload, D)
    elif wl["mode"] == "async":
        line = run_async(args, wl, args.workload, D)
    else:
        dl = None
        if wl.get("delayed"):
            def dl(w):
                return args.tc_us * (1 + args.slow) if w == 0 else args.tc_us
        line = run_ours(args, wl, args.workload, D, delay_us=dl, e2e=not args.no_e2e)
        if D.n == 1 and line is not None and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(wl, D.n, budget_s=args.cpu_budget)
        if D.n > 1 and args.workload == "r50x8" and not args.no_extras:
            ex = extras(args, D)
            if line is not None:
                line["extras"] = ex
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
