#!/usr/bin/env python3
"""Reference peel_approx / peel_exact outcomes on the config graphs
(tests/golden/peel_configs.json), from the UNMODIFIED reference
(oracle/_ref/libkclique_ref.so).  Minutes per entry on 8 cores.

    python tools/make_peel_config_goldens.py --entries 2:4:approx 1:3:exact
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402,F401

from paper_2002_10047_b200 import gen  # noqa: E402
from tests import reforacle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "peel_configs.json")

ap = argparse.ArgumentParser()
ap.add_argument("--entries", nargs="+", default=["2:4:approx"])
ap.add_argument("--threads", type=int, default=0)
ap.add_argument("--eps", type=float, default=0.5)
a = ap.parse_args()
R = reforacle.Ref()
if a.threads:
    R.set_threads(a.threads)
out = json.load(open(OUT)) if os.path.exists(OUT) else {}
for ent in a.entries:
    cid, k, mode = ent.split(":")
    cid, k, exact = int(cid), int(k), mode == "exact"
    key = f"config{cid}_k{k}_{mode}"
    if key in out:
        continue
    spec = gen.CONFIGS[cid]
    g = gen.load_config_graph(cid)
    rg = R.graph(g)
    r, _, _ = R.rank(rg, g.n, spec["strategy"], spec["eps"], 0)
    dg, _ = R.direct(rg, r)
    o = R.peel(rg, dg, g.n, k, exact, a.eps)
    e = {"config": cid, "k": k, "exact": exact, "eps": a.eps, "strategy": spec["strategy"],
         "strategy_eps": spec["eps"], "graph_digest": g.digest(), "rounds": o["rounds"],
         "total_cliques": str(o["total_cliques"]), "best_round": o["best_round"],
         "best_density": o["best_density"].hex(), "num_dense": int(len(o["dense_vertices"])),
         "dense_digest": f"{gen.digest_u32(o['dense_vertices']):016x}",
         "ref_seconds": o["seconds"], "threads": R.max_threads()}
    if exact:
        e["core_digest"] = f"{gen.digest_u64(o['core']):016x}"
    out[key] = e
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(key, e, flush=True)
    R.dg_destroy(dg)
    R.graph_destroy(rg)
