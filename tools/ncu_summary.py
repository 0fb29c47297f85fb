#!/usr/bin/env python3
"""One line per kernel launch of an ncu report: duration, DRAM / L2 / SM
throughput, IPC, occupancy, and DRAM bytes.

    python tools/ncu_summary.py REPORT.ncu-rep [--json OUT]
"""
import argparse
import csv
import io
import json
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("report")
ap.add_argument("--json")
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
want = {
    "dur_ns": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_pct": "lts__t_sectors.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "ipc": "sm__inst_executed.avg.per_cycle_active",
    "occ": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1_hit": "l1tex__t_sector_hit_rate.pct",
    "l2_hit": "lts__t_sector_hit_rate.pct",
    "inst": "smsp__inst_executed.sum",
    "thr_per_inst": "smsp__thread_inst_executed_per_inst_executed.ratio",
}
idx = {k: hdr.index(v) for k, v in want.items() if v in hdr}
units = rows[1]
scale = {"ms": 1e6, "us": 1e3, "ns": 1.0, "s": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9,
         "byte": 1.0}
ni = hdr.index("Kernel Name")
res = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    d = {"kernel": r[ni][:60]}
    for k, i in idx.items():
        try:
            d[k] = float(r[i].replace(",", "")) * scale.get(units[i], 1.0)
        except ValueError:
            d[k] = r[i]
    res.append(d)
    print(f"{d['kernel'][:44]:44s} {d.get('dur_ns',0)/1e6:8.3f} ms dram {d.get('dram_pct','?'):>6} "
          f"l2 {d.get('l2_pct','?'):>6} sm {d.get('sm_pct','?'):>6} ipc {d.get('ipc','?'):>5} "
          f"occ {d.get('occ','?'):>6} thr/inst {d.get('thr_per_inst','?'):>5} "
          f"dramMB {(d.get('dram_read',0)+d.get('dram_write',0))/1e6:9.1f}")
if a.json:
    json.dump(res, open(a.json, "w"), indent=1)
