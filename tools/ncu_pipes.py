#!/usr/bin/env python3
"""Per-launch pipe / memory-unit utilisation and stall breakdown from an ncu
--set full report (which unit bounds a kernel).

    python tools/ncu_pipes.py REPORT.ncu-rep [--launch N] [--grep SUBSTR]
"""
import argparse
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("report")
ap.add_argument("--launch", type=int, default=None)
ap.add_argument("--grep", default="")
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
for li, r in enumerate(rows[2:]):
    if a.launch is not None and li != a.launch:
        continue
    d = dict(zip(hdr, r))
    name = d.get("Kernel Name", "")[:60]
    print(f"== [{li}] {name} {d.get('gpu__time_duration.sum')} ms")
    items = []
    for k, v in d.items():
        if a.grep and a.grep not in k:
            continue
        try:
            fv = float(v)
        except ValueError:
            continue
        if ("pipe_" in k and "pct_of_peak_sustained_active" in k and "inst_executed" in k) or \
           ("warp_issue_stalled" in k and k.endswith("per_warp_active.pct")) or \
           ("wavefronts" in k and k.endswith(".sum")) or \
           k in ("sm__inst_executed.sum", "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                 "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
                 "smsp__issue_active.avg.pct_of_peak_sustained_active"):
            if fv != 0:
                items.append((k, fv))
    for k, v in sorted(items, key=lambda x: -x[1])[:60]:
        print(f"   {v:14.3f}  {k}")
