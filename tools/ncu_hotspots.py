#!/usr/bin/env python3
"""Ranks CUDA source lines of one kernel launch in an ncu report by warp-
stall samples (needs -lineinfo builds and --import-source on).

    python tools/ncu_hotspots.py REPORT.ncu-rep --skip N [--top 30]
"""
import argparse
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("report")
ap.add_argument("--skip", type=int, default=0, help="launch index within the report")
ap.add_argument("--top", type=int, default=30)
a = ap.parse_args()

out = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv",
                      "--print-source=cuda,sass", "--launch-skip", str(a.skip),
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
si = hdr.index("Warp Stall Sampling (All Samples)")
ii = hdr.index("Instructions Executed")
ti = hdr.index("Avg. Threads Executed")
stall_cols = [(i, n[6:]) for i, n in enumerate(hdr) if n.startswith("stall_") and "Not Issued" not in n]
lines = []
for r in rows:
    if not r or not r[0].isdigit() or len(r) <= si:
        continue
    try:
        s = int(r[si])
    except ValueError:
        continue
    st = sorted(((n, int(r[i])) for i, n in stall_cols if r[i] not in ("", "-", "0")),
                key=lambda x: -x[1])[:3]
    lines.append((s, int(r[ii] or 0), r[ti], r[0], r[1].strip(), st))
tot = sum(x[0] for x in lines) or 1
print(f"total samples {tot}")
for s, n, thr, ln, src, st in sorted(lines, reverse=True)[:a.top]:
    print(f"{100*s/tot:5.1f}% inst={n:>11} thr={thr:>3} L{ln:>4} {src[:64]:64s} "
          + " ".join(f"{k}={v}" for k, v in st))
