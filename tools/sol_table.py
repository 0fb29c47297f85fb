#!/usr/bin/env python3
"""Folds the speed-of-light sweep (tools/sol_sweep.sh) into one row per
(config, k): counting-kernel time, time-weighted SM throughput (% of peak
issue), DRAM and L2 bytes, and the B_alg-based HBM fraction.

    python tools/sol_table.py gpurun_out/sol [--json profiles/...json]
"""
import csv
import glob
import json
import os
import sys

d = sys.argv[1]
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    "MEASURED_PEAKS.json") else 6546.2
rows = []
for f in sorted(glob.glob(os.path.join(d, "*.csv"))):
    data = list(csv.reader(open(f)))
    hdr = None
    per = {}
    for r in data:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            x = dict(zip(hdr, r))
            v = float(x["Metric Value"].replace(",", ""))
            per.setdefault(x["ID"], {})[x["Metric Name"]] = v
    if not per:
        continue
    t = sum(p["gpu__time_duration.sum"] for p in per.values())
    sm = sum(p["gpu__time_duration.sum"] * p["sm__throughput.avg.pct_of_peak_sustained_elapsed"]
             for p in per.values()) / t
    dram = sum(p["dram__bytes_read.sum"] + p["dram__bytes_write.sum"] for p in per.values())
    l2 = sum(p["lts__t_bytes.sum"] for p in per.values())
    inst = sum(p["sm__inst_executed.sum"] for p in per.values())
    rows.append({"case": os.path.basename(f)[:-4], "launches": len(per), "ncu_ms": t / 1e6,
                 "issue_frac": sm / 100.0, "dram_gb": dram / 1e9, "l2_gb": l2 / 1e9,
                 "dram_gbs": dram / t, "l2_gbs": l2 / t, "warp_inst_g": inst / 1e9})
for r in rows:
    print(f"{r['case']:8s} {r['launches']:3d} launches {r['ncu_ms']:9.2f} ms  issue {r['issue_frac']:.2f}"
          f"  DRAM {r['dram_gb']:7.2f} GB ({r['dram_gbs']:7.1f} GB/s)  L2 {r['l2_gb']:8.2f} GB"
          f" ({r['l2_gbs']:7.1f} GB/s)  {r['warp_inst_g']:8.2f} G warp-inst")
if len(sys.argv) > 3 and sys.argv[2] == "--json":
    json.dump(rows, open(sys.argv[3], "w"), indent=1)
