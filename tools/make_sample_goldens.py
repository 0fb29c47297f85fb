#!/usr/bin/env python3
"""Writes tests/golden/sample_cases.json: colorful_sparsify digests and
approx_count results of the UNMODIFIED reference (proj/src/sampling.cpp,
compiled into oracle/_ref/libkclique_ref.so) on seeded graphs, plus
analytic_variance values.

    python tools/make_sample_goldens.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2002_10047_b200 import gen  # noqa: E402
from tests import reforacle  # noqa: E402

R = reforacle.Ref()
R.set_threads(8)
OUT = os.path.join(ROOT, "tests", "golden", "sample_cases.json")
cases = []
graphs = [("gnp", [40, 0.4, 9], gen.gnp(40, 0.4, 9)),
          ("rmat", [12, 1 << 15, 7, 1], gen.rmat(12, 1 << 15, seed=7, permute=True)),
          ("rmat", [14, 1 << 18, 11, 0], gen.rmat(14, 1 << 18, seed=11, permute=False)),
          ("config", [2], gen.load_config_graph(2))]
for kind, params, g in graphs:
    rg = R.graph(g)
    for colors, seed in [(1, 0), (2, 5), (3, 17), (8, 123456789)]:
        off, adj = R.colorful_sparsify(rg, g.n, colors, seed)
        ent = {"graph": {"kind": kind, "params": params, "digest": g.digest(), "n": g.n},
               "colors": colors, "seed": seed, "m": int(len(adj) // 2),
               "digest": f"{gen.digest_u64(off):016x}:{gen.digest_u32(adj):016x}",
               "approx": {}}
        for k, strat, eps in [(3, 0, 1.0), (4, 0, 1.0), (4, 4, 0.5), (5, 2, 1.0)]:
            if kind == "config" and k == 5:
                continue
            a = R.approx_count(rg, k, colors, seed, strat, eps)
            ent["approx"][f"{k}:{strat}:{eps}"] = {"sub_count": str(a["sub_count"]),
                                                   "p": a["p"].hex(),
                                                   "estimate": a["estimate"].hex()}
        cases.append(ent)
        print(kind, params, colors, seed, ent["m"], flush=True)
    R.graph_destroy(rg)
var = []
for tc, p, k, pairs in [(1000, 0.5, 4, [0, 0, 30, 7]), (12345, 0.125, 5, [0, 0, 100, 50, 3]),
                        (7, 1.0, 3, [0, 0, 2]), (0, 0.3, 2, [])]:
    var.append({"true_count": tc, "p": p, "k": k, "pairs": pairs,
                "variance": R.analytic_variance(tc, p, k, pairs).hex()})
with open(OUT, "w") as f:
    json.dump({"cases": cases, "variance": var}, f, indent=0)
print("wrote", OUT)
