#!/usr/bin/env python3
"""Shared-memory wavefronts per CUDA source line of one launch in an ncu
report (the LSU data pipe is the counting kernels' busiest unit):

    python tools/ncu_smem_lines.py REPORT.ncu-rep --skip N [--top 25]
"""
import argparse
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("report")
ap.add_argument("--skip", type=int, default=0)
ap.add_argument("--top", type=int, default=25)
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv",
                      "--print-source=cuda,sass", "--launch-skip", str(a.skip),
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
wi = hdr.index("L1 Wavefronts Shared")
ii = hdr.index("L1 Wavefronts Shared Ideal")
lines = []
for r in rows:
    if not r or not r[0].isdigit() or len(r) <= wi:
        continue
    try:
        w, ideal = int(r[wi] or 0), int(r[ii] or 0)
    except ValueError:
        continue
    if w:
        lines.append((w, ideal, r[0], r[1].strip()))
tot = sum(x[0] for x in lines) or 1
print(f"total shared wavefronts {tot}")
for w, ideal, ln, src in sorted(lines, reverse=True)[:a.top]:
    print(f"{100*w/tot:5.1f}% wf={w:>11} ideal={ideal:>11} L{ln:>4} {src[:80]}")
