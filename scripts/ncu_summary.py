#!/usr/bin/env python3
"""Summarize an ncu report (--set full) into a markdown table of the metrics the roofline uses.

    python scripts/ncu_summary.py gpurun_out/r01/prof.ncu-rep [--algo-bytes B] > profiles/x.md
"""
import argparse
import csv
import io
import subprocess

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("nvlrx__bytes.sum", "NVLink rx bytes"),
    ("nvltx__bytes.sum", "NVLink tx bytes"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "stall long scoreboard"),
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--algo-bytes", type=float, nargs="*", default=None,
                    help="algorithmic bytes per launch, in launch order")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print(f"ncu report `{a.report}` (--set full, --clock-control none; cold-cache, serialized replay)\n")
    cols = ["kernel"] + [label for m, label in METRICS if m in hdr] + ["DRAM GB/s", "algorithmic GB/s"]
    print("| " + " | ".join(cols) + " |")
    print("|" + "---|" * len(cols))
    for li, r in enumerate(rows[2:]):
        vals = {m: (r[hdr.index(m)], units[hdr.index(m)]) for m, _ in METRICS if m in hdr}
        name = r[hdr.index("Kernel Name")]
        name = name.split("::")[-1].split("(")[0]
        out = [name]
        for m, label in METRICS:
            if m in vals:
                v, u = vals[m]
                out.append(f"{v} {u}".strip())

        def num(m):
            v, u = vals.get(m, ("0", "byte"))
            try:
                return float(v.replace(",", "")) * SCALE.get(u, 1)
            except ValueError:
                return 0.0
        dur = num("gpu__time_duration.sum")
        dram = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
        out.append(f"{dram / dur / 1e9:.1f}" if dur else "-")
        if a.algo_bytes and li < len(a.algo_bytes):
            out.append(f"{a.algo_bytes[li] / dur / 1e9:.1f}")
        else:
            out.append("-")
        print("| " + " | ".join(out) + " |")


if __name__ == "__main__":
    main()
