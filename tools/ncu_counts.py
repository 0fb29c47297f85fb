#!/usr/bin/env python3
"""ncu counters of the counting kernels of one (config, k) count, reduced to a
JSON entry (run on the GPU box; profiles/ncu_summary.json keeps the entries
bench.py quotes as `traffic` and `limiter`).

    python tools/ncu_counts.py --config 2 --k 4 [--pv] --out gpurun_out/ncu_c2k4.json
"""
import argparse
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "lts__t_bytes.sum", "smsp__inst_executed.sum",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "smsp__thread_inst_executed_per_inst_executed.ratio",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
           "lts__t_sectors.avg.pct_of_peak_sustained_elapsed",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed"]

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, required=True)
ap.add_argument("--k", type=int, default=4)
ap.add_argument("--pv", action="store_true")
ap.add_argument("--out", required=True)
a = ap.parse_args()
if a.config == 5:
    cmd = [sys.executable, os.path.join(ROOT, "tools", "prof_c5.py"), "5", "pv" if a.pv else "total"]
else:
    cmd = [sys.executable, os.path.join(ROOT, "tools", "prof_count.py"), "--config", str(a.config),
           "--k", str(a.k), "--reps", "1"] + (["--pv"] if a.pv else [])
log = a.out + ".csv"
ncu = ["ncu", "--metrics", ",".join(METRICS), "--clock-control", "none", "-k", "regex:count_",
       "--csv", "--log-file", log] + cmd
subprocess.run(ncu, check=True, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
hdr, launches = None, {}
for r in csv.reader(open(log)):
    if hdr is None:
        if r and r[0] == "ID":
            hdr = r
        continue
    d = dict(zip(hdr, r))
    e = launches.setdefault(int(d["ID"]), {"kernel": d["Kernel Name"][:90], "grid": d["Grid Size"],
                                           "block": d["Block Size"]})
    e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
# endpoint_count_kernel belongs to the device graph build, not to the count
L = [v for _, v in sorted(launches.items()) if "endpoint_count" not in v["kernel"]]
T = sum(v["gpu__time_duration.sum"] for v in L)


def tw(m):
    return sum(v[m] * v["gpu__time_duration.sum"] for v in L) / T


out = {
    "source": "ncu --metrics ... --clock-control none -k regex:count_ on " + " ".join(cmd[1:]),
    "kernels_per_count": len(L),
    "ncu_duration_ns_sum": T,
    "dram_bytes_per_launch": sum(v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"] for v in L),
    "l2_bytes_per_launch": sum(v["lts__t_bytes.sum"] for v in L),
    "warp_inst": sum(v["smsp__inst_executed.sum"] for v in L),
    "lsu_wavefront_pct_time_weighted": tw("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed"),
    "lsu_shared_wavefront_pct_time_weighted":
        tw("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    "issue_active_pct_time_weighted": tw("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "threads_per_inst_time_weighted": tw("smsp__thread_inst_executed_per_inst_executed.ratio"),
    "l2_pct_time_weighted": tw("lts__t_sectors.avg.pct_of_peak_sustained_elapsed"),
    "dram_pct_time_weighted": tw("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
    "launches": [{
        "kernel": v["kernel"], "grid": v["grid"], "block": v["block"],
        "dur_ns": v["gpu__time_duration.sum"],
        "dram_bytes": v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"],
        "l2_bytes": v["lts__t_bytes.sum"], "warp_inst": v["smsp__inst_executed.sum"],
        "lsu_wavefront_pct": v["l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed"],
        "issue_active_pct": v["smsp__issue_active.avg.pct_of_peak_sustained_active"],
        "occupancy_pct": v["sm__warps_active.avg.pct_of_peak_sustained_active"],
        "thr_per_inst": v["smsp__thread_inst_executed_per_inst_executed.ratio"],
    } for v in L],
}
json.dump(out, open(a.out, "w"), indent=1)
os.remove(log)
print(a.out, "kernels", len(L), "ms %.2f" % (T / 1e6), "lsu %.1f%% issue %.1f%%" % (
    out["lsu_wavefront_pct_time_weighted"], out["issue_active_pct_time_weighted"]))
