"""Every intra-GPU kernel variant stays parity-green, not only the default one.

The variant is chosen once per process from the environment (RP_PREDUCE_TMA for fp32 replicas,
RP_PREDUCE_BF16 for bf16 replicas: 0 = LDG/STG kernel, 1-4 = CTA-synchronous TMA pipelines,
5/6 = warp-specialized with a static tile split, 7 = warp-specialized with dynamic tile
scheduling, the default for launches of >= RP_DYN_MIN_BYTES = 1 GiB), so each case re-runs the
bit-exact kernel tests in a subprocess.
"""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{"RP_PREDUCE_TMA": "0"}, {"RP_PREDUCE_TMA": "3"}, {"RP_PREDUCE_TMA": "5"},
                                 {"RP_PREDUCE_TMA": "6"}, {"RP_PREDUCE_TMA": "7", "RP_WS_K8": "2"},
                                 # variant 7 on every launch (by default launches under 1 GiB take 5/6)
                                 {"RP_PREDUCE_TMA": "7", "RP_PREDUCE_BF16": "7", "RP_DYN_MIN_BYTES": "0"},
                                 {"RP_PREDUCE_BF16": "5"}, {"RP_PREDUCE_BF16": "6"}])
def test_kernel_variant_parity(env):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu",
           os.path.join(ROOT, "tests", "test_gpu_kernels.py"), os.path.join(ROOT, "tests", "test_gpu_parity.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env={**os.environ, **env})
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-2000:]
