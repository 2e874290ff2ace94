"""bench.py's host-side arithmetic (no GPU): workload layouts and the roofline fractions computed
from per-launch records."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_default_workload_spreads_eight_workers(bench):
    wl = bench.WORKLOADS["r50x8"]
    assert [bench.wpg_of(wl, n) for n in (1, 2, 4, 8)] == [8, 4, 2, 1]   # configs[1] ... configs[2]
    assert wl["scaling"] == "strong" and wl["n"] == bench.N_R50 and wl["k"] == 3
    with pytest.raises(SystemExit):
        bench.wpg_of(wl, 3)
    assert bench.wpg_of(bench.WORKLOADS["cfg4"], 8) == 2                  # configs[3]: 16 workers on 8


def _rec(ms, nvl, batch, cross=True, hbm=0):
    return {"ms": ms, "bytes_nvlink": nvl, "bytes_hbm": hbm, "batch": batch, "cross": cross}


def test_cross_roofline_bottleneck_and_step_level(bench):
    peak = bench.NVLINK_PEAK * 1e9
    # two steps on two GPUs; step 0: rank 0 moves 2 GB in 4 ms (rank 1: 1 GB, waits 4 ms),
    # step 1: rank 1 is the bottleneck (3 GB in 5 ms)
    recs = [[_rec(4.0, 2e9, 0), _rec(5.0, 1e9, 1)], [_rec(4.0, 1e9, 0), _rec(5.0, 3e9, 1)]]
    ms_total = 10.0
    r = bench.cross_roofline(recs, ms_total, 2, {"hbm_gbs": 6543.4}, "measured", None)
    # bottleneck GPU per step: (2 GB + 3 GB) / (4 ms + 5 ms)
    assert r["achieved"] == pytest.approx(5e9 / 9e-3 / 1e9, rel=1e-3)
    assert r["frac"] == pytest.approx(5e9 / 9e-3 / peak, rel=1e-3)
    # kernel level: all bytes / all kernel time
    assert r["kernel_level"]["achieved"] == pytest.approx(7e9 / 18e-3 / 1e9, rel=1e-3)
    # step level: sum_t max bytes / peak over the measured time
    assert r["step_level"]["frac"] == pytest.approx((2e9 + 3e9) / peak / 10e-3, rel=1e-3)
    assert r["busiest_gpu"]["rank"] == 1 and r["launches"] == 4


def test_cross_roofline_ignores_intra_launches_and_reports_missing_counters(bench):
    recs = [[_rec(1.0, 0, 0, cross=False, hbm=6e9), _rec(2.0, 1e9, 0)], [_rec(2.0, 1e9, 0)]]
    r = bench.cross_roofline(recs, 2.0, 1, {"hbm_gbs": 6543.4}, "measured", [{"error": "x"}, {"error": "x"}])
    assert r["launches"] == 2 and r["traffic"]["unavailable"] == ["x"]
    h = bench.hbm_roofline(recs, {"hbm_gbs": 6543.4}, "measured", "none", 2)
    assert h["achieved"] == pytest.approx(6e9 / 1e-3 / 1e9) and h["launches"] == 1
    assert bench.cross_roofline([[_rec(1.0, 0, 0, cross=False)]], 1.0, 1, {}, "", None) is None
