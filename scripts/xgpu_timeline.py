#!/usr/bin/env python3
"""Analyse the cross-GPU kernel item timeline dumped with RP_XGPU_PROFILE=path (files path.<rank>).

Each record: t_start, t_ready (wait satisfied), t_end (flag posted) in %globaltimer ns, meta.
"""
import sys

import numpy as np

KIND = {0: "A", 1: "B", 2: "C"}


def cta_breakdown(path):
    """RP_XGPU_PROFILE=path also dumps path.cta.<rank>: per CTA ns [ring wait, signal wait, flag wait, total]."""
    import os
    base, rank = path.rsplit(".", 1)
    p = f"{base}.cta.{rank}"
    if not os.path.exists(p):
        return
    raw = np.fromfile(p, dtype=np.uint64)
    a = raw[:4 * 2048].reshape(-1, 4).astype(np.float64)
    if raw.size >= 6 * 2048:   # absolute begin / end per CTA (warp-specialized kernel)
        be = raw[4 * 2048:6 * 2048].reshape(-1, 2)
        be = be[be[:, 1] > 0].astype(np.float64)
        if len(be):
            t0 = be[:, 0].min()
            b, e = (be[:, 0] - t0) / 1e3, (be[:, 1] - t0) / 1e3
            q = np.percentile(e, [0, 10, 50, 90, 100])
            print(f"  CTA work begins within {b.max():.1f} us of the first; CTA end times (us after the first "
                  f"begin) min/p10/p50/p90/max = " + "/".join(f"{v:.1f}" for v in q))
    a = a[a[:, 3] > 0]
    if not len(a):
        return
    tot = a[:, 3].sum()
    ring, sig, flag = (a[:, i].sum() / tot for i in range(3))
    print(f"  per-CTA time ({len(a)} CTAs, mean total {a[:, 3].mean() / 1e3:.1f} us): [0] {ring:.1%}, [1] {sig:.1%}, "
          f"[2] peer-flag wait {flag:.1%}, rest {1 - ring - sig - flag:.1%}  (register kernel: [0] smem-ring wait, [1] "
          f"signal wait; warp-specialized kernel: [0] consumer warp 0 waiting for loaded data, [1] its signal wait, "
          f"[2] the producer's flag waits)")


def sig_timeline(path, bin_us=10.0):
    """Per-iteration view (warp-specialized kernel): SIG times and producer flag waits over the kernel."""
    import os
    base, rank = path.rsplit(".", 1)
    p = f"{base}.cta.{rank}"
    if not os.path.exists(p):
        return
    raw = np.fromfile(p, dtype=np.uint64)
    SIG, WAIT = 32, 32
    sb = 6 * 2048
    wb = sb + 2048 * SIG
    cb = wb + 2048 * 2 * WAIT
    if raw.size < cb + 2 * 2048:
        return
    be = raw[4 * 2048:6 * 2048].reshape(-1, 2)
    live = np.nonzero(be[:, 1] > 0)[0]
    if not len(live):
        return
    t0 = be[live, 0].min()
    span = (be[live, 1].max() - t0) / 1e3
    print(f"  [{rank}] kernel: first CTA begin at globaltimer {int(t0)} ns, last CTA end +{span:.1f} us")
    cnt = raw[cb:cb + 2 * 2048].reshape(-1, 2)
    sig = raw[sb:wb].reshape(2048, SIG)
    rows = []
    for c in live:
        ns = int(min(cnt[c, 0], SIG))
        rows.append([((int(v) & ~3) - int(t0)) / 1e3 for v in sig[c, :ns]])
    kmax = max(len(r) for r in rows)
    line = []
    for k in range(kmax):
        v = np.array([r[k] for r in rows if len(r) > k])
        line.append(f"{k}:{np.percentile(v, 50):.0f}({len(v)})")
    print("  SIG k: median us after kernel begin (CTAs reaching it): " + " ".join(line))
    wt = raw[wb:cb].reshape(2048, WAIT, 2)
    nb = int(span // bin_us) + 1
    busy = {0: np.zeros(nb), 1: np.zeros(nb), 2: np.zeros(nb)}
    tot = {0: 0.0, 1: 0.0, 2: 0.0}
    for c in live:
        nw = int(min(cnt[c, 1], WAIT))
        for q in range(nw):
            k = int(wt[c, q, 0]) & 3
            a = ((int(wt[c, q, 0]) & ~3) - int(t0)) / 1e3
            b = (int(wt[c, q, 1]) - int(t0)) / 1e3
            tot[k] += b - a
            i = int(a // bin_us)
            while a < b and i < nb:
                e = min(b, (i + 1) * bin_us)
                busy[k][i] += e - a
                a, i = e, i + 1
    names = {0: "A-flag", 1: "B-flag", 2: "READY"}
    n = len(live)
    for k in (2, 0, 1):
        if tot[k] > 0:
            prof = " ".join(f"{x / (n * bin_us):.2f}" for x in busy[k])
            print(f"  {names[k]} waits: {tot[k] / n:.1f} us per CTA; fraction of CTAs waiting per {bin_us:.0f} us bin: {prof}")
    ends = np.sort((be[live, 1] - t0) / 1e3)
    act = " ".join(f"{(ends > (i + 1) * bin_us).mean():.2f}" for i in range(nb))
    print(f"  fraction of CTAs still running at the end of each bin: {act}")


def main():
    for path in sys.argv[1:]:
        cta_breakdown(path)
        sig_timeline(path)
        rec = np.fromfile(path, dtype=np.uint64).reshape(-1, 4)
        rec = rec[rec[:, 0] > 0]
        if not len(rec):  # the warp-specialized kernel records only the per-CTA breakdown
            print(f"== {path}: no item records")
            continue
        t0 = rec[:, 0].min()
        ts, tr, te = [(rec[:, i] - t0).astype(np.float64) / 1e3 for i in range(3)]  # us
        kind = (rec[:, 3] >> np.uint64(62)).astype(int)
        cta = ((rec[:, 3] >> np.uint64(32)) & np.uint64(0xFFFFFF)).astype(int)
        print(f"== {path}: {len(rec)} items, kernel span {te.max():.1f} us, CTAs {cta.max() + 1}")
        for k in (0, 1, 2):
            m = kind == k
            if not m.any():
                continue
            wait = tr[m] - ts[m]
            work = te[m] - tr[m]
            print(f"  {KIND[k]}: n={m.sum():5d}  first start {ts[m].min():8.1f}  last end {te[m].max():8.1f}  "
                  f"wait mean {wait.mean():7.2f} max {wait.max():7.2f}  work mean {work.mean():7.2f} "
                  f"p50 {np.median(work):7.2f} max {work.max():7.2f} us")
        span = te.max()
        bucket = max(10.0, span / 15)
        print(f"  t(us)   work-A  work-B  work-C  waiting   (CTAs busy, averaged per {bucket:.0f} us bucket)")
        t = 0.0
        while t < span:
            lo, hi = t, t + bucket

            def occ(a, z):
                return np.clip(np.minimum(z, hi) - np.maximum(a, lo), 0, None).sum() / bucket
            line = [occ(tr[kind == k], te[kind == k]) for k in (0, 1, 2)] + [occ(ts, tr)]
            print(f"  {lo:7.0f}  " + "  ".join(f"{v:6.1f}" for v in line))
            t += bucket


if __name__ == "__main__":
    main()
