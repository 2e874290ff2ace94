"""Seeded synthetic inputs shared by the oracle and the tests.

This package holds ONLY the counter-based random generator that produces the
synthetic parameter and gradient vectors. It contains none of the method's
arithmetic (no SGD, no averaging, no scheduling). The CUDA side implements the
same generator independently (``paper_1909_08029_b200/csrc/xi.cu``); a GPU
test checks the two bit for bit.
"""
from .gen import (  # noqa: F401
    SEED_X,
    SEED_G,
    mix64,
    key64,
    xi,
    x0,
    grad,
)
