#!/usr/bin/env python3
"""Config 5 (R-MAT s24, degree order) counting profile: device-built graph,
k = 4 totals and per-vertex counts with the count statistics."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_10047_b200 import gen, kcg  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["total", "pv"]
p = gen.CONFIGS[cfg]["rmat"]
with kcg.DeviceGraph.rmat(p["scale"], p["samples"], seed=p["seed"], permute=p["permute"]) as h:
    h.rank(gen.CONFIGS[cfg]["strategy"], gen.CONFIGS[cfg]["eps"], download=False)
    h.direct(download=False)
    for mode in modes:
        t, _ = h.count(4, per_vertex=mode == "pv")
        tm = h.timings()
        print(mode, t, f"count_ms={tm['count_ms']:.1f} kernel_ms={tm['count_kernel_ms']:.1f}",
              h.count_stats(), flush=True)
