#!/usr/bin/env python3
"""Folds a per-launch ncu summary (tools/ncu_summary.py --json) of ONE
counting call into profiles/ncu_summary.json under `key`: DRAM bytes of the
call (roofline.traffic in bench.py) and the issue-side evidence -- the
time-weighted SM throughput (% of peak issue) and IPC of its launches.

    python tools/ncu_entry.py gpurun_out/c2full_summary.json config2_k4 "<how>"
"""
import json
import os
import sys

src, key, how = sys.argv[1], sys.argv[2], sys.argv[3]
rows = json.load(open(src))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
out = json.load(open(out_path)) if os.path.exists(out_path) else {}
t = sum(r["dur_ns"] for r in rows)
w = lambda f: sum(r[f] * r["dur_ns"] for r in rows) / t  # noqa: E731
out[key] = {
    "dram_bytes_per_launch": sum(r["dram_read"] + r["dram_write"] for r in rows),
    "kernels_per_count": len(rows),
    "ncu_duration_ns_sum": t,
    "sm_throughput_pct_time_weighted": w("sm_pct"),
    "ipc_time_weighted": w("ipc"),
    "issue_slot_peak_ipc": 4.0,
    "threads_per_inst_time_weighted": w("thr_per_inst"),
    "dram_pct_time_weighted": w("dram_pct"),
    "l2_pct_time_weighted": w("l2_pct"),
    "launches": [{k: r[k] for k in ("kernel", "dur_ns", "sm_pct", "ipc", "occ", "dram_pct",
                                    "l2_pct", "thr_per_inst")} | {
        "dram_bytes": r["dram_read"] + r["dram_write"]} for r in rows],
    "source": how,
}
json.dump(out, open(out_path, "w"), indent=1)
print(key, {k: v for k, v in out[key].items() if k != "launches"})
