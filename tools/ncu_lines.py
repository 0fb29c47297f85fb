#!/usr/bin/env python3
"""Per-source-line instruction and stall-sample totals of one kernel in an
.ncu-rep (ncu --page source --print-source cuda,sass --csv), largest first.
usage: ncu_lines.py REPORT KERNEL_ID_SPEC [TOP]   (spec e.g. ::regex:count_cta:2)"""
import csv
import io
import subprocess
import sys

rep, spec = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-id", spec], capture_output=True, text=True).stdout
fname, hdr, cur, agg = None, None, None, {}
seen = {}  # SASS address -> (priority, line key): inlined frames list one instruction under several lines


def prio(f):
    return 2 if f.endswith(".cuh") else 1 if f.endswith(".cu") else 0



for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    if r[0]:
        cur = (fname, int(r[0]), r[1])
        agg.setdefault(cur, [0, 0, 0, 0])
        continue
    if r[2] == "...":
        continue
    d = dict(zip(hdr[2:], r[2:]))
    vals = [int(d["Instructions Executed"] or 0), int(d["# Samples"] or 0),
            int(d["Thread Instructions Executed"] or 0), int(d["L1 Wavefronts Shared"] or 0)]
    addr = r[2]
    if addr in seen and seen[addr][0] >= prio(cur[0]):
        continue
    if addr in seen:
        old = agg[seen[addr][1]]
        for i in range(4):
            old[i] -= vals[i]
    seen[addr] = (prio(cur[0]), cur)
    a = agg[cur]
    for i in range(4):
        a[i] += vals[i]
ti = sum(a[0] for a in agg.values())
ts = sum(a[1] for a in agg.values())
print(f"total warp inst {ti}  samples {ts}")
for (f, ln, src), a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{f}:{ln:<5} inst {100*a[0]/ti:5.1f}%  smp {100*a[1]/max(ts,1):5.1f}%  thr/inst {a[2]/max(a[0],1):4.1f}  ldsw {a[3]:>10}  {src.strip()[:80]}")
