"""Small runs of the hot kernels for compute-sanitizer (SURVEY §4 tier v: racecheck, synccheck).

    RP_DYN_MIN_BYTES=0 compute-sanitizer --tool racecheck python scripts/sanitize_case.py

(a) the intra-GPU dynamic-tile TMA kernel (preduce_dyn_kernel; RP_DYN_MIN_BYTES=0 selects it at a
small size), 8 workers, GB + GD k = 3; (b) the cross-GPU kernel for 2 and 3 emulated GPUs in one
cooperative launch (RP_FLAG_EMULATE: flags, staging, TMA bulk pushes between the virtual GPUs),
each checked bit for bit against the oracle so a silent corruption also fails the run.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import sim  # noqa: E402
from paper_1909_08029_b200.runner import LockstepRunner  # noqa: E402


def check(r, world, n, T, wpg, **kw):
    r.synchronize()
    X, _ = sim.run_lockstep(world, n, T, workers_per_gpu=wpg, **kw)
    for w in range(world):
        got = r.x(w).cpu().numpy()
        if not np.array_equal(got.view(np.uint32), X[w].view(np.uint32)):
            raise SystemExit(f"worker {w}: differs from the oracle")
    r.close()


def main():
    T = 3
    n = 300_007
    r = LockstepRunner(8, n, mode="gd", group_size=3, c_thres=4, seed_gd=3)
    r.run(T)
    check(r, 8, n, T, 8, mode="gd", k=3, c_thres=4, seed_gd=3)
    print("intra-GPU kernel ok", flush=True)
    n = 200_003
    r = LockstepRunner(4, n, mode="static", rule="shift_k", group_size=3, n_gpus=2, device=0, emulate=True)
    r.run(T)
    check(r, 4, n, T, 2, mode="static", rule="shift_k", k=3)
    print("cross-GPU kernel (2 emulated GPUs, m <= 2) ok", flush=True)
    r = LockstepRunner(3, n, mode="gd", group_size=3, n_gpus=3, device=0, emulate=True)
    r.run(T)
    check(r, 3, n, T, 1, mode="gd", k=3)
    print("cross-GPU kernel (3 emulated GPUs, kp = 3) ok", flush=True)


if __name__ == "__main__":
    main()
