"""A few lockstep steps of the cross-GPU kernel on ONE GPU (RP_FLAG_EMULATE), for ncu:

    ncu --set full -k regex:xgpu_ws_emul -c 2 python scripts/emul_case.py [V] [wpg] [n]

V virtual GPUs, wpg workers each, static SHIFT_K(V*wpg, V*wpg) = one group of everybody, so
every step runs the A, B and C stages of every virtual GPU in one cooperative launch.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_08029_b200.runner import LockstepRunner  # noqa: E402


def main():
    V = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    wpg = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 25_557_032
    world = V * wpg
    r = LockstepRunner(world, n, mode="static", rule="shift_k", group_size=world, n_gpus=V, device=0,
                       grad_mode="resident", emulate=True)
    r.run_native(4)
    r.synchronize()
    st = r.ctx.stats()
    r.close()
    print(f"emulated {V} GPUs x {wpg} workers, n={n}: {st['cross_gpu_groups']} cross groups, "
          f"{st['kernel_launches']} launches")


if __name__ == "__main__":
    main()
