import os
import sys
from fractions import Fraction

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: longer CPU test")


def pytest_collection_modifyitems(config, items):
    # `pytest tests` on a machine without CUDA: gpu-marked tests skip instead of failing with
    # RP_ENODEV (the driver selects them explicitly with -m gpu on a B200)
    import torch
    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="needs a CUDA device (gpu marker)")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def golden_lines(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return [ln.rstrip("\n") for ln in f if ln.strip() and not ln.startswith("#")]


def golden_matrix(name):
    return [[Fraction(tok) for tok in ln.split()] for ln in golden_lines(name)]


@pytest.fixture(scope="session")
def gpu_available():
    import torch
    return torch.cuda.is_available()
