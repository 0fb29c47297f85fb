#!/usr/bin/env python3
"""Writes tests/golden/kcore_cases.json: the UNMODIFIED reference's
rank_by_kcore (orientation.cpp:23-46, a sequential (degree, id) heap order)
on seeded graphs -- rank digests, and the ranks themselves for small n.

    python tools/make_kcore_goldens.py
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
cases = []


def add(kind, params, g):
    rg = R.graph(g)
    r, _, _ = R.rank(rg, g.n, gen.KCORE, 1.0, 0)
    R.graph_destroy(rg)
    e = {"kind": kind, "params": params, "digest": g.digest(), "n": g.n,
         "rank_digest": f"{gen.digest_u32(r):016x}"}
    if g.n <= 200:
        e["rank"] = r.tolist()
    cases.append(e)


for seed in range(40):
    n = 5 + seed % 40
    add("gnp", [n, [0.1, 0.3, 0.6][seed % 3], seed + 7100],
        gen.gnp(n, [0.1, 0.3, 0.6][seed % 3], seed + 7100))
for s, e, seed, perm in [(10, 8192, 3, 0), (12, 1 << 15, 7, 1), (14, 1 << 18, 5, 1)]:
    add("rmat", [s, e, seed, perm], gen.rmat(s, e, seed=seed, permute=bool(perm)))
add("config", [1], gen.load_config_graph(1))
with open(os.path.join(ROOT, "tests", "golden", "kcore_cases.json"), "w") as f:
    json.dump({"cases": cases}, f)
print("wrote", len(cases), "cases")
