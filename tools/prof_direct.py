#!/usr/bin/env python3
"""Profiling driver for ranking + DAG build on a config graph:
`reps` x (rank, direct) on the handle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_10047_b200 import gen, kcg  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
spec = gen.CONFIGS[cfg]
if "rmat" in spec:  # bit-identical device generator (configs 2, 5)
    p = spec["rmat"]
    h = kcg.DeviceGraph.rmat(p["scale"], p["samples"], seed=p["seed"], permute=p["permute"])
else:
    h = kcg.DeviceGraph.from_graph(gen.load_config_graph(cfg, cache=False))
with h:
    for _ in range(reps):
        h.rank(gen.gpu_strategy(spec), spec["eps"], download=False)
        r = h.timings()["rank_ms"]
        h.direct(download=False)
        print(f"rank_ms={r:.3f} direct_ms={h.timings()['direct_ms']:.3f}", flush=True)
