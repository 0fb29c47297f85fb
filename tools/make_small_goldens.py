#!/usr/bin/env python3
"""Writes tests/golden/small_cases.json: small seeded graphs with the
outputs of the UNMODIFIED reference library (oracle/_ref/libkclique_ref.so)
— rankings (+rounds, alpha), DAG digests, totals and per-vertex counts.

The GPU parity tests compare libkcg against these fixtures (the compiled
reference does not exist on the GPU box).  Run in the build container:

    python tools/make_small_goldens.py
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


def hexd(x):
    return f"{x:016x}"


def graph_entry(g, edges=None):
    e = {"n": g.n, "m": g.m, "digest": g.digest()}
    if edges is not None:
        e["edges"] = np.asarray(edges, dtype=np.int64).reshape(-1).tolist()
    return e


def rank_block(rg, g, strategies):
    out = {}
    for name, strat, eps in strategies:
        r, rounds, _ = R.rank(rg, g.n, strat, eps, 0)
        dg, _ = R.direct(rg, r)
        off, adj = R.dg_csr(dg, g.n, g.m)
        R.dg_destroy(dg)
        ent = {"strategy": strat, "eps": eps, "rounds": rounds,
               "max_out": int(np.diff(off).max()) if g.n else 0,
               "dag_digest": f"{hexd(gen.digest_u64(off))}:{hexd(gen.digest_u32(adj))}",
               "rank_digest": hexd(gen.digest_u32(r))}
        if g.n <= 64:
            ent["rank"] = r.tolist()
        if strat == gen.BARENBOIM_ELKIN:
            ent["alpha"] = R.estimate_arboricity(rg, eps)
        out[name] = ent
    return out


def counts_block(rg, g, ks, pv_ks, strat=gen.DEGREE, eps=1.0, brute=False):
    r, _, _ = R.rank(rg, g.n, strat, eps, 0)
    dg, _ = R.direct(rg, r)
    out = {}
    for k in ks:
        if brute:
            total, pv = R.brute_force(rg, g.n, k)
        else:
            total, pv, _ = R.count(dg, g.n, k, want_pv=k in pv_ks)
        ent = {"total": str(total)}
        if k in pv_ks:
            if g.n <= 64:
                ent["pv"] = [int(x) for x in pv]
            ent["pv_digest"] = hexd(gen.digest_u64(pv))
        out[str(k)] = ent
    R.dg_destroy(dg)
    return out


ALL = [("degree", 0, 1.0), ("original", 1, 1.0), ("goodrich_pszona", 3, 1.0),
       ("barenboim_elkin", 4, 1.0), ("barenboim_elkin_eps05", 4, 0.5)]


def main():
    cases = []
    # acceptance criterion 3 battery (proj/tests/acceptance.cpp:156-217)
    for seed in range(200):
        n = 5 + seed % 26
        p = [0.2, 0.4, 0.6][seed % 3]
        g = gen.gnp(n, p, seed + 31000)
        rg = R.graph(g)
        ks = list(range(2, 8))
        cases.append({"name": f"accept3_s{seed}", "kind": "gnp", "params": [n, p, seed + 31000],
                      "graph": graph_entry(g), "rankings": rank_block(rg, g, ALL),
                      "counts": counts_block(rg, g, ks, ks, brute=True)})
        R.graph_destroy(rg)
    print("accept3 done", flush=True)
    # R-MAT scale 12: CTA tier (out-degree > 32) under degree and BE orders
    g = gen.rmat(12, 1 << 15, seed=7, permute=True)
    rg = R.graph(g)
    cases.append({"name": "rmat12", "kind": "rmat", "params": [12, 1 << 15, 7, 1],
                  "graph": graph_entry(g),
                  "rankings": rank_block(rg, g, ALL),
                  "counts": counts_block(rg, g, [2, 3, 4, 5, 6], [3, 4, 5]),
                  "counts_be05": counts_block(rg, g, [4, 5], [4], gen.BARENBOIM_ELKIN, 0.5)})
    R.graph_destroy(rg)
    print("rmat12 done", flush=True)
    rng = np.random.default_rng(11)
    # heavy tier: vertex 0 adjacent to 1500 vertices, identity order
    base = gen.rmat(11, 1 << 14, seed=11, permute=True)
    e = [(u, int(v)) for u in range(base.n) for v in
         base.adj[base.offsets[u]:base.offsets[u + 1]] if u < v]
    hub = rng.choice(np.arange(1, base.n), 1500, replace=False)
    e += [(0, int(x)) for x in hub]
    g = gen.from_edges(base.n, np.array(e))
    rg = R.graph(g)
    cases.append({"name": "hub1500", "kind": "edges", "graph": graph_entry(g, e),
                  "rankings": rank_block(rg, g, ALL[:1]),
                  "counts_original": counts_block(rg, g, [3, 4, 5], [3, 4, 5], gen.ORIGINAL)})
    R.graph_destroy(rg)
    # planted 50-clique: candidate sets above 32 and deep recursion
    n = 400
    e = set()
    members = rng.choice(n, 50, replace=False)
    for i in range(50):
        for j in range(i + 1, 50):
            a, b = int(members[i]), int(members[j])
            e.add((min(a, b), max(a, b)))
    while len(e) < 1225 + 1600:
        a, b = (int(x) for x in rng.integers(0, n, 2))
        if a != b:
            e.add((min(a, b), max(a, b)))
    e = sorted(e)
    g = gen.from_edges(n, np.array(e))
    rg = R.graph(g)
    cases.append({"name": "planted50", "kind": "edges", "graph": graph_entry(g, e),
                  "rankings": rank_block(rg, g, ALL[:1] + ALL[3:4]),
                  "counts": counts_block(rg, g, [3, 4, 5, 6, 7], [3, 4, 5, 6])})
    R.graph_destroy(rg)
    print("planted50 done", flush=True)
    # planted 36-clique: large k (generic explicit-stack path)
    n = 120
    e = set()
    members = rng.choice(n, 36, replace=False)
    for i in range(36):
        for j in range(i + 1, 36):
            a, b = int(members[i]), int(members[j])
            e.add((min(a, b), max(a, b)))
    while len(e) < 630 + 240:
        a, b = (int(x) for x in rng.integers(0, n, 2))
        if a != b:
            e.add((min(a, b), max(a, b)))
    e = sorted(e)
    g = gen.from_edges(n, np.array(e))
    rg = R.graph(g)
    cases.append({"name": "planted36", "kind": "edges", "graph": graph_entry(g, e),
                  "rankings": rank_block(rg, g, ALL[:1]),
                  "counts": counts_block(rg, g, [4, 5, 30, 33, 34, 35, 36, 37], [33, 36])})
    R.graph_destroy(rg)
    print("planted36 done", flush=True)
    path = os.path.join(ROOT, "tests", "golden", "small_cases.json")
    with open(path, "w") as f:
        json.dump({"generator": "tools/make_small_goldens.py",
                   "oracle": "oracle/_ref/libkclique_ref.so (unmodified reference)",
                   "cases": cases}, f, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
