"""Multi-GPU parity (one process per GPU, cross-GPU groups over NVLink peer memory) vs the oracle.

Runs only when the box exposes >= 2 GPUs (gpurun --gpus 2/4); each case launches torchrun.
"""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N_R50 = 25_557_032


def _ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(nproc, spec, timeout=600, script="multi_gpu_worker.py", env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", script), json.dumps(spec)]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT,
                       env={**os.environ, **(env or {})})
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-4000:]
    assert p.stdout.count("OK") == nproc, p.stdout


CASES = [
    # (gpus, wpg, n, k, mode, rule, steps, sample)
    (2, 1, (1 << 20) + 3, 2, "static", "shift_k", 20, 0),     # one cross pair per step, ragged
    (2, 2, 100_003, 3, "static", "shift_k", 12, 0),           # pre-reduction of co-resident members
    (2, 4, 100_003, 3, "gd", None, 12, 0),                    # GB+GD: several cross parts per GPU
    (2, 1, 5, 2, "static", "shift_k", 6, 0),                  # slices smaller than a tile
    (2, 1, 1, 2, "static", "shift_k", 4, 0),                  # scalar-only
    (2, 2, 65_536, 2, "static", "paper4", 8, 0),              # PAPER4 2 nodes x 2
    (2, 1, N_R50, 2, "gd", None, 4, 4099),                    # ResNet-50 size, sampled
    (4, 1, 200_003, 3, "gd", None, 10, 0),                    # cfg 3 shape at 4 GPUs
    (4, 2, 200_003, 3, "static", "shift_k", 10, 0),           # cfg 4 shape at 4 GPUs
    (4, 4, 60_001, 4, "static", "paper4", 8, 0),              # PAPER4 4 nodes x 4 (fig:schedule)
    (8, 1, 200_003, 3, "gd", None, 10, 0),                    # cfg 3 shape at 8 GPUs
    (8, 2, 100_003, 3, "static", "shift_k", 10, 0),           # cfg 4 shape at 8 GPUs
    (8, 8, 20_011, 3, "gd", None, 6, 0),                      # 64 workers: 8 cross parts per GPU
    (2, 4, 50_007, 3, "gd+ii", None, 8, 0),                   # Inter-Intra (§5.2), GPU = node
    (4, 8, 30_011, 3, "gd+ii", None, 8, 0),                   # configs[1] layout, Inter-Intra
]


@pytest.mark.parametrize("gpus,extra", [(2, dict(wpg=2, n=60_011, k=3, mode="static", rule="shift_k", steps=10,
                                                 momentum=[0.9, 1e-4])),
                                        (2, dict(wpg=4, n=30_001, k=3, mode="gd", steps=9, momentum=[0.9, 1e-4],
                                                 section_length=2)),
                                        (4, dict(wpg=2, n=40_003, k=3, mode="gd", steps=8, momentum=[0.9, 1e-4],
                                                 ii=True))])
def test_multi_gpu_momentum_section_length(gpus, extra):
    # P:1274 momentum + weight decay fused into the cross-GPU kernel (buffers stay per worker);
    # P:1312 section length; Inter-Intra groups
    if _ngpu() < gpus:
        pytest.skip(f"needs {gpus} GPUs")
    _run(gpus, {"sample": 0, "rule": None, **extra})


@pytest.mark.parametrize("gpus,wpg,n,k,mode,rule,steps,sample", CASES)
def test_multi_gpu_parity(gpus, wpg, n, k, mode, rule, steps, sample):
    if _ngpu() < gpus:
        pytest.skip(f"needs {gpus} GPUs")
    ii = mode == "gd+ii"
    _run(gpus, dict(wpg=wpg, n=n, k=k, mode="gd" if ii else mode, rule=rule, steps=steps, sample=sample, ii=ii))


ASYNC_CASES = [
    # (gpus, wpg, n, k, c_thres, steps)
    (2, 2, 50_003, 3, 2, 10),        # cfg 5 shape at 2 GPUs: shared GG, slowed worker 0
    (2, 1, 40_000, 2, 0, 12),        # AD-PSGD-like pairs, filter off
    (4, 2, 30_011, 3, 4, 8),         # cfg 5 shape at 4 GPUs
]


@pytest.mark.parametrize("gpus,wpg,n,k,c_thres,steps", ASYNC_CASES)
def test_multi_gpu_async_shared_gg_replay(gpus, wpg, n, k, c_thres, steps, tmp_path):
    if _ngpu() < gpus:
        pytest.skip(f"needs {gpus} GPUs")
    _run(gpus, dict(wpg=wpg, n=n, k=k, c_thres=c_thres, steps=steps, tmp=str(tmp_path)),
         script="multi_gpu_async_worker.py")


NVLS_CASES = [
    # (gpus, spec): NVLS P-Reduce (rp_nvls_enable). kp = 2 groups are bit-exact
    # (fp32 addition of two partials is commutative); kp >= 3 groups sum in the switch's order
    # (reading R25) and are held to the north-star bound 1e-6 * max|x| (tol).
    (2, dict(wpg=1, n=(1 << 20) + 3, k=2, mode="static", rule="shift_k", steps=20, nvls=2)),
    (2, dict(wpg=2, n=100_003, k=3, mode="static", rule="shift_k", steps=12, nvls=2)),
    (2, dict(wpg=4, n=100_003, k=3, mode="gd", steps=12, nvls=2)),
    (2, dict(wpg=1, n=5, k=2, mode="static", rule="shift_k", steps=6, nvls=2)),
    (2, dict(wpg=1, n=1, k=2, mode="static", rule="shift_k", steps=4, nvls=2)),
    (2, dict(wpg=2, n=60_011, k=3, mode="static", rule="shift_k", steps=10, nvls=2, momentum=[0.9, 1e-4])),
    (2, dict(wpg=1, n=N_R50, k=2, mode="gd", steps=4, sample=4099, nvls=2)),
    (4, dict(wpg=1, n=200_003, k=3, mode="gd", steps=20, nvls=3, tol=1e-6)),
    (4, dict(wpg=2, n=200_003, k=3, mode="static", rule="shift_k", steps=20, nvls=2, tol=1e-6)),
    (4, dict(wpg=4, n=60_001, k=4, mode="static", rule="paper4", steps=8, nvls=3, tol=1e-6)),
    (4, dict(wpg=8, n=30_011, k=3, mode="gd", steps=10, nvls=2, tol=1e-6)),
]


@pytest.mark.parametrize("gpus,spec", NVLS_CASES)
def test_multi_gpu_nvls_parity(gpus, spec):
    if _ngpu() < gpus:
        pytest.skip(f"needs {gpus} GPUs")
    _run(gpus, {"sample": 0, "rule": None, **spec})


@pytest.mark.parametrize("gpus,split,spec", [
    # RP_XGPU_SPLIT caps the cross launch's grid beside a concurrent intra-GPU launch; uncapped (0)
    # and capped grids on different GPUs must still agree on every chunk flag (the chunk
    # geometry depends on n and kp only)
    (2, "0", dict(wpg=4, n=50_007, k=3, mode="gd", steps=8, ii=True)),
    (2, "0", dict(wpg=4, n=100_003, k=3, mode="gd", steps=12)),
    (2, "37", dict(wpg=4, n=50_007, k=3, mode="gd", steps=8, ii=True)),
    (4, "37", dict(wpg=8, n=30_011, k=3, mode="gd", steps=8, ii=True)),
])
def test_multi_gpu_split_modes(gpus, split, spec):
    if _ngpu() < gpus:
        pytest.skip(f"needs {gpus} GPUs")
    _run(gpus, {"sample": 0, "rule": None, **spec}, env={"RP_XGPU_SPLIT": split})


@pytest.mark.parametrize("gpus,env,spec", [
    # geometry knobs (RP_XGPU_ITERS / RP_XGPU_MIN_TILES): one lane iteration, many small chunks
    (2, {"RP_XGPU_ITERS": "1"}, dict(wpg=2, n=300_007, k=3, mode="static", rule="shift_k", steps=8)),
    (2, {"RP_XGPU_ITERS": "16", "RP_XGPU_MIN_TILES": "1"}, dict(wpg=4, n=3_000_017, k=3, mode="gd", steps=8)),
])
def test_multi_gpu_geometry_knobs(gpus, env, spec):
    if _ngpu() < gpus:
        pytest.skip(f"needs {gpus} GPUs")
    _run(gpus, {"sample": 0, "rule": None, **spec}, env=env)


@pytest.mark.parametrize("gpus,spec", [
    # RP_DEBUG_POISON: owners' staging rows NaN-filled before every cross launch (race check)
    (2, dict(wpg=4, n=300_007, k=3, mode="gd", steps=12)),
    (2, dict(wpg=2, n=200_003, k=3, mode="static", rule="shift_k", steps=10, dtype="bf16")),
    (4, dict(wpg=1, n=500_009, k=3, mode="gd", steps=12)),
    (4, dict(wpg=2, n=300_007, k=3, mode="static", rule="shift_k", steps=9, momentum=[0.9, 1e-4])),
])
def test_multi_gpu_poisoned_staging(gpus, spec):
    if _ngpu() < gpus:
        pytest.skip(f"needs {gpus} GPUs")
    _run(gpus, {"sample": 0, "rule": None, **spec}, env={"RP_DEBUG_POISON": "1"})


BF16_CASES = [
    # bf16 replicas across GPUs (reading R26): fp32 partials over NVLink, the mean rounded once
    # to bf16 and pushed as bf16; bit-exact vs the oracle's fused_group_update_bf16
    (2, dict(wpg=1, n=(1 << 20) + 3, k=2, mode="static", rule="shift_k", steps=12)),
    (2, dict(wpg=2, n=100_003, k=3, mode="static", rule="shift_k", steps=10)),
    (2, dict(wpg=4, n=100_001, k=3, mode="gd", steps=10)),
    (2, dict(wpg=4, n=50_007, k=3, mode="gd", steps=8, ii=True)),
    (2, dict(wpg=1, n=5, k=2, mode="static", rule="shift_k", steps=6)),
    (2, dict(wpg=1, n=4102, k=2, mode="static", rule="shift_k", steps=6)),   # odd bf16 vector count
    (4, dict(wpg=2, n=200_003, k=3, mode="gd", steps=10)),
    (4, dict(wpg=8, n=30_011, k=3, mode="gd", steps=8, ii=True)),
]


@pytest.mark.parametrize("gpus,spec", BF16_CASES)
def test_multi_gpu_bf16_parity(gpus, spec):
    if _ngpu() < gpus:
        pytest.skip(f"needs {gpus} GPUs")
    _run(gpus, {"sample": 0, "rule": None, "dtype": "bf16", **spec})


@pytest.mark.parametrize("gpus,spec", [
    # rp_lockstep_run (the native step loop) across GPUs, resident gradients
    (2, dict(wpg=4, n=100_003, k=3, mode="gd", steps=12)),
    (2, dict(wpg=4, n=50_007, k=3, mode="gd", steps=10, ii=True)),
    (2, dict(wpg=2, n=100_003, k=3, mode="static", rule="shift_k", steps=10)),
    (4, dict(wpg=8, n=30_011, k=3, mode="gd", steps=8, ii=True)),
    (4, dict(wpg=1, n=200_003, k=3, mode="gd", steps=10, dtype="bf16")),
    # the bench's default problem at N = 2 (8 workers, ResNet-50 size, GB + GD), 100 steps
    (2, dict(wpg=4, n=N_R50, k=3, mode="gd", steps=100, sample=4099)),
    # configs[2] at N = 4 (kp = 3 groups), 100 steps
    (4, dict(wpg=1, n=N_R50, k=3, mode="gd", steps=100, sample=4099)),
])
def test_multi_gpu_native_executor(gpus, spec):
    if _ngpu() < gpus:
        pytest.skip(f"needs {gpus} GPUs")
    _run(gpus, {"sample": 0, "rule": None, "native": True, **spec})


def test_multi_gpu_watchdog_reports_timeout():
    # a peer that never arrives: the flag wait gives up after watchdog_s, the kernel ends, the
    # host call returns RP_ETIMEOUT and the CUDA context stays usable (no __trap)
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    _run(2, {}, script="multi_gpu_watchdog_worker.py", timeout=300)
