#!/usr/bin/env python3
"""One-line summaries of bench JSON files."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads([ln for ln in open(f) if ln.startswith("{")][0])
    except Exception as e:  # noqa: BLE001
        print(f, "ERR", e)
        continue
    r = d.get("roofline") or {}
    o = r.get("other_kernel") or {}
    x = r if r.get("bound") == "nvlink" else o
    sl = (x.get("step_level") or {}).get("frac")
    kl = (x.get("kernel_level") or {}).get("frac")
    print(f"{f}: {d.get('impl')} value={d['value']} ms/step={d['ms_per_step']} "
          f"roof={r.get('bound')}:{r.get('achieved')}({r.get('frac')}) other={o.get('bound')}:{o.get('achieved')} "
          f"nvlink kernel-level={kl} step-level={sl} busbw={d.get('busbw_gbs')}")
