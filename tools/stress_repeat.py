#!/usr/bin/env python3
"""Repeats counts on one resident DAG and checks that every repetition gives
the same total and the same per-vertex digest (a race in the staging or
credit paths would show up as a flicker).  GPU box only.

    python tools/stress_repeat.py CONFIG K REPS [pv]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_10047_b200 import gen, kcg  # noqa: E402

cfg, k, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
pv = len(sys.argv) > 4 and sys.argv[4] == "pv"
spec = gen.CONFIGS[cfg]
if "rmat" in spec:
    p = spec["rmat"]
    h = kcg.DeviceGraph.rmat(p["scale"], p["samples"], seed=p["seed"], permute=p["permute"])
else:
    h = kcg.DeviceGraph.from_graph(gen.load_config_graph(cfg, cache=False))
with h:
    h.rank(gen.gpu_strategy(spec), spec["eps"], download=False)
    h.direct(download=False)
    seen = set()
    for _ in range(reps):
        t, v = h.count(k, per_vertex=pv)
        seen.add((t, gen.digest_u64(v) if pv else 0))
    print(f"config {cfg} k={k} pv={pv} reps={reps} distinct results: {len(seen)}", sorted(seen)[:2])
    sys.exit(0 if len(seen) == 1 else 1)
