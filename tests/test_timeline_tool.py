"""scripts/xgpu_timeline.py reads the RP_XGPU_PROFILE per-CTA dump whose layout rp_internal.h
defines (kCtaSig / kCtaWait / kCtaStatWords): the two must agree, and the per-iteration view must
read a synthetic dump back (CPU only)."""
import importlib.util
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _tool():
    spec = importlib.util.spec_from_file_location("xgpu_timeline", os.path.join(ROOT, "scripts", "xgpu_timeline.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def _layout():
    h = open(os.path.join(ROOT, "paper_1909_08029_b200", "csrc", "rp_internal.h")).read()
    sig = int(re.search(r"kCtaSig = (\d+)", h).group(1))
    wait = int(re.search(r"kCtaWait = (\d+)", h).group(1))
    assert "kCtaSigBase = 6 * 2048" in h
    return sig, wait


def test_dump_layout_matches_header(tmp_path, capsys):
    SIG, WAIT = _layout()
    sb = 6 * 2048
    wb = sb + 2048 * SIG
    cb = wb + 2048 * 2 * WAIT
    raw = np.zeros(cb + 2 * 2048, dtype=np.uint64)
    t0 = 1_000_000_000
    for c, (b, e) in enumerate([(0, 50_000), (1_000, 60_000)]):   # two CTAs, ns after t0
        raw[4 * 2048 + 2 * c] = t0 + b
        raw[4 * 2048 + 2 * c + 1] = t0 + e
        raw[cb + 2 * c] = 2                                          # two SIGs each
        raw[sb + SIG * c + 0] = ((t0 + 10_000) & ~3) | 1             # posts A flags
        raw[sb + SIG * c + 1] = ((t0 + 30_000) & ~3) | 2             # posts B flags
        raw[cb + 2 * c + 1] = 1                                      # one A-flag wait of 5 us
        raw[wb + 2 * WAIT * c] = ((t0 + 20_000) & ~3) | 0
        raw[wb + 2 * WAIT * c + 1] = t0 + 25_000
    raw[:4 * 2048].reshape(-1, 4)[:2, 3] = 50_000
    base = tmp_path / "tl"
    raw.tofile(f"{base}.cta.0")
    _tool().sig_timeline(f"{base}.0")
    out = capsys.readouterr().out
    assert "last CTA end +60.0 us" in out
    assert "0:10(2) 1:30(2)" in out                                  # SIG medians, CTAs reaching them
    assert "A-flag waits: 5.0 us per CTA" in out
    assert "READY" not in out and "B-flag" not in out
