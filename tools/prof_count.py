#!/usr/bin/env python3
"""Profiling driver: one config graph, rank + direct, then `reps` counts.
Used under ncu (tools/README in DESIGN.md §Profiling):

    python tools/prof_count.py --config 2 --k 4 --reps 2
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2002_10047_b200 import gen, kcg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--k", type=int, default=4)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--pv", action="store_true")
a = ap.parse_args()
spec = gen.CONFIGS[a.config]
g = gen.load_config_graph(a.config, cache=False)
with kcg.DeviceGraph.from_graph(g) as h:
    h.rank(gen.gpu_strategy(spec), spec["eps"], download=False)
    h.direct(download=False)
    for _ in range(a.reps):
        t, _ = h.count(a.k, per_vertex=a.pv)
    tm = h.timings()
    print(f"config {a.config} k={a.k} total={t} count_ms={tm['count_ms']:.3f} "
          f"kernel_ms={tm['count_kernel_ms']:.3f} stats={h.count_stats()}")
