#!/usr/bin/env python3
"""Times the UNMODIFIED reference (oracle/_ref/libkclique_ref.so) on this
machine's host cores for the config/k pairs that finish in minutes:
make_ranking, direct_by_ranking and count_total with default_parallelism,
as the CLI's PhaseTimer does (kclique_main.cpp:33-45,153-184).  One JSON
line per (config, k).

    python tools/ref_box_times.py [--out FILE]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_10047_b200 import gen  # noqa: E402
from tests import reforacle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=None)
ap.add_argument("--pairs", nargs="*", default=["1:3", "1:4", "2:4", "2:5", "3:4", "3:5", "3:6",
                                                 "4:6"])
a = ap.parse_args()
R = reforacle.Ref()
R.set_threads(os.cpu_count() or 1)
graphs = {}
for pair in a.pairs:
    cid, k = map(int, pair.split(":"))
    spec = gen.CONFIGS[cid]
    if cid not in graphs:
        graphs[cid] = gen.load_config_graph(cid, cache=False)
    g = graphs[cid]
    rg = R.graph(g)
    t0 = time.perf_counter()
    rank, _, t_rank = R.rank(rg, g.n, spec["strategy"], spec["eps"], 0)
    dg, t_dir = R.direct(rg, rank)
    total, _, t_count = R.count(dg, g.n, k, parallelism=2)  # default_parallelism(k)
    rec = {"config": cid, "k": k, "total": str(total), "threads": R.max_threads(),
           "rank_s": t_rank, "direct_s": t_dir, "count_s": t_count,
           "step_s": time.perf_counter() - t0}
    R.dg_destroy(dg)
    R.graph_destroy(rg)
    line = json.dumps(rec)
    print(line, flush=True)
    if a.out:
        with open(a.out, "a") as f:
            f.write(line + "\n")
