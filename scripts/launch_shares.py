#!/usr/bin/env python3
"""Per-kernel launch count, mean device time and share of total from an ncu --csv launch list."""
import collections
import csv
import sys

lines = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[1:]:
    agg.setdefault(r[ki].split("(")[0], []).append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
print("| kernel | launches | mean us | share of device time |\n|---|---|---|---|")
for k, v in agg.items():
    print(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot * 100:.1f}% |")
