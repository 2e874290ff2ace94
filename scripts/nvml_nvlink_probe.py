"""Which NVML NVLink byte counters move, and by how much, for a known peer transfer?

Round 2, first box: every nvmlDeviceGetFieldValues NVLink counter (THROUGHPUT_*, COUNT_*_BYTES,
per link and aggregate) answered NVML_ERROR_NOT_SUPPORTED on the B200 boxes (driver 580). This
probe therefore reads the GPU Performance Monitoring (GPM) NVLink metrics around 4 x 1 GiB copies
GPU0 -> GPU1 and prints them next to the bytes moved. bench.py uses the same GPM metrics
(paper_1909_08029_b200/nvlink_counters.py) around its timed region.
"""
import os
import sys
import time

import pynvml
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_08029_b200.nvlink_counters import GpmNvlink  # noqa: E402


def smi(args):
    import subprocess
    try:
        return subprocess.run(["nvidia-smi"] + args, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:  # noqa: BLE001
        return f"nvidia-smi failed: {e}"


def main():
    pynvml.nvmlInit()
    for i in range(2):
        h = pynvml.nvmlDeviceGetHandleByIndex(i)
        for name, fn in (("streaming enabled", lambda: pynvml.nvmlGpmQueryIfStreamingEnabled(h)),
                         ("enable streaming", lambda: pynvml.nvmlGpmSetStreamingEnabled(h, 1))):
            try:
                print(f"GPU{i} {name}: {fn()}")
            except Exception as e:  # noqa: BLE001
                print(f"GPU{i} {name}: {e}")
    print("nvidia-smi nvlink -gt d (before):")
    print(smi(["nvlink", "-gt", "d", "-i", "0"])[:3000])
    mons = [GpmNvlink(i) for i in range(2)]
    for i, m in enumerate(mons):
        print(f"GPU{i}: GPM supported={m.supported} ({m.why})")
    nbytes = 1 << 30
    a = torch.empty(nbytes // 4, device="cuda:0")
    b = torch.empty(nbytes // 4, device="cuda:1")
    a.uniform_()
    b.copy_(a)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    for rep in range(2):
        for m in mons:
            m.start()
        t0 = time.perf_counter()
        for _ in range(4):
            b.copy_(a)
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        dt = time.perf_counter() - t0
        res = [m.stop() for m in mons]
        print(f"rep {rep}: moved {4 * nbytes} bytes GPU0 -> GPU1 in {dt * 1e3:.2f} ms "
              f"({4 * nbytes / dt / 1e9:.1f} GB/s)")
        for i, r in enumerate(res):
            print(f"  GPU{i}: {r}")
    print("nvidia-smi nvlink -gt d (after 8 GiB GPU0 -> GPU1):")
    print(smi(["nvlink", "-gt", "d", "-i", "0"])[:3000])
    print(smi(["nvlink", "-gt", "d", "-i", "1"])[:3000])


if __name__ == "__main__":
    main()
