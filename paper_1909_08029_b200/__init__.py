"""B200-native Partial All-Reduce (Ripples, arXiv 1909.08029) — Python binding.

The compute path lives in ``librp.so`` (CUDA kernels for sm_100a + a C++
engine behind the C ABI of ``include/rp.h``). This package only marshals
arguments; it never computes the method itself and has no CPU fallback.
"""
from .rp import (  # noqa: F401
    RP_OK, RP_EINVAL, RP_ESTATE, RP_EPROTO, RP_ECONFLICT, RP_ETIMEOUT, RP_ECUDA, RP_ENOMEM,
    RP_ENODEV, RP_EAGAIN, RP_SCHED_PAPER4, RP_SCHED_SHIFT_K, RP_WAIT_DEVICE, RP_MAX_GROUP, RP_MAX_WORLD,
    RP_FLAG_TRACE, RP_FLAG_TIMING, RP_FLAG_SHARED_GG, RP_FLAG_RANDOM_GG, RP_FLAG_INTER_INTRA, RP_FLAG_EMULATE, RP_FLAG_GRAPH, RPError, rp_timing, rp_peer_info, rp_config, rp_group, rp_stats, load_library, library_path,
    Context, fill_xi, compute_delay, EXPORTED_SYMBOLS,
)
