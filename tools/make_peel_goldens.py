#!/usr/bin/env python3
"""Writes tests/golden/peel_cases.json: outputs of the UNMODIFIED reference
peeling code (proj/src/peeling.cpp, compiled into
oracle/_ref/libkclique_ref.so by oracle/Makefile) on seeded graphs:

* update sequences: random batches until every vertex is peeled, each step
  with the reference's removed / changed / updated counts
  (the shape of test_peeling.cpp:101-148, own batches);
* peel_exact and peel_approx outcomes (rounds, total, best round, density,
  core and dense-vertex digests / arrays) on small and mid-size graphs,
  including the tiered counting cases and config 1.

Run in the build container:  python tools/make_peel_goldens.py
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
OUT = os.path.join(ROOT, "tests", "golden", "peel_cases.json")


def hexd(x):
    return f"{x:016x}"


def oriented(g, strat=gen.DEGREE, eps=1.0):
    rg = R.graph(g)
    r, _, _ = R.rank(rg, g.n, strat, eps, 0)
    dg, _ = R.direct(rg, r)
    return rg, dg


def close(rg, dg):
    R.dg_destroy(dg)
    R.graph_destroy(rg)


def update_case(spec, g, k, seed):
    rg, dg = oriented(g)
    _, pv, _ = R.count(dg, g.n, k, want_pv=True)
    counts = pv.astype(np.uint64).copy()
    peeled = np.zeros(g.n, np.uint8)
    rng = np.random.default_rng(seed)
    alive = list(range(g.n))
    steps = []
    while alive:
        rng.shuffle(alive)
        take = 1 + int(rng.integers(0, min(len(alive), 4)))
        batch = sorted(alive[:take])
        alive = alive[take:]
        removed, changed = R.update_counts(rg, dg, g.n, k, counts, batch, peeled)
        peeled[batch] = 1
        steps.append({"batch": batch, "removed": removed, "changed": changed.tolist(),
                      "counts": counts.tolist()})
    close(rg, dg)
    return {"graph": spec, "k": k, "initial": pv.tolist(), "steps": steps}


def peel_case(spec, g, k, exact, eps=0.5, strat=gen.DEGREE, strat_eps=1.0):
    rg, dg = oriented(g, strat, strat_eps)
    o = R.peel(rg, dg, g.n, k, exact, eps)
    close(rg, dg)
    ent = {"graph": spec, "k": k, "exact": bool(exact), "eps": eps, "strategy": strat,
           "strategy_eps": strat_eps, "rounds": o["rounds"],
           "total_cliques": str(o["total_cliques"]), "best_round": o["best_round"],
           "best_density": o["best_density"].hex(),
           "num_dense": int(len(o["dense_vertices"])),
           "dense_digest": hexd(gen.digest_u32(o["dense_vertices"]))}
    if exact:
        ent["core_digest"] = hexd(gen.digest_u64(o["core"]))
    if g.n <= 64:
        ent["dense_vertices"] = o["dense_vertices"].tolist()
        if exact:
            ent["core"] = o["core"].tolist()
    print(f"  peel {spec['kind']} {spec.get('params')} k={k} exact={exact}: rounds "
          f"{o['rounds']} density {o['best_density']:.4f} ({o['seconds']:.2f}s)", flush=True)
    return ent


def spec_of(kind, params, g, edges=None):
    s = {"kind": kind, "params": params, "digest": g.digest(), "n": g.n, "m": g.m}
    if edges is not None:
        s["edges"] = np.asarray(edges, dtype=np.int64).reshape(-1).tolist()
    return s


def main():
    out = {"updates": [], "peels": []}
    # update sequences
    for seed in range(10):
        g = gen.gnp(12, 0.45, seed + 2200)
        spec = spec_of("gnp", [12, 0.45, seed + 2200], g)
        for k in (2, 3, 4):
            out["updates"].append(update_case(spec, g, k, seed * 31 + 5 + k))
    g = gen.gnp(40, 0.5, 77)
    spec = spec_of("gnp", [40, 0.5, 77], g)
    for k in (3, 5):
        out["updates"].append(update_case(spec, g, k, 4242 + k))
    # peeling outcomes
    for seed in range(14):
        n = 8 + seed % 7
        g = gen.gnp(n, 0.5, seed + 5100)
        spec = spec_of("gnp", [n, 0.5, seed + 5100], g)
        for k in (3, 4):
            for exact in (True, False):
                out["peels"].append(peel_case(spec, g, k, exact))
    g = gen.gnp(30, 0.35, 808)
    spec = spec_of("gnp", [30, 0.35, 808], g)
    for exact in (True, False):
        out["peels"].append(peel_case(spec, g, 4, exact))
        out["peels"].append(peel_case(spec, g, 4, exact, strat=gen.BARENBOIM_ELKIN,
                                      strat_eps=0.5))
    two = np.array([[0, 1], [1, 2], [0, 2], [3, 4], [4, 5], [3, 5]])
    g = gen.from_edges(6, two)
    spec = spec_of("edges", None, g, two)
    out["peels"].append(peel_case(spec, g, 3, True))
    path = np.array([[i, i + 1] for i in range(7)])
    g = gen.from_edges(8, path)
    spec = spec_of("edges", None, g, path)
    out["peels"].append(peel_case(spec, g, 3, False))
    out["peels"].append(peel_case(spec, g, 2, True))
    for s, e, seed, perm in [(10, 8192, 3, 0), (12, 1 << 15, 7, 1)]:
        g = gen.rmat(s, e, seed=seed, permute=bool(perm))
        spec = spec_of("rmat", [s, e, seed, perm], g)
        for k in (3, 4):
            for exact in (True, False):
                out["peels"].append(peel_case(spec, g, k, exact))
    for eps in (0.1, 1.0):
        g = gen.rmat(12, 1 << 15, seed=7, permute=True)
        spec = spec_of("rmat", [12, 1 << 15, 7, 1], g)
        out["peels"].append(peel_case(spec, g, 5, False, eps=eps))
    g = gen.load_config_graph(1)
    spec = {"kind": "config", "params": [1], "digest": g.digest(), "n": g.n, "m": g.m}
    for exact in (True, False):
        out["peels"].append(peel_case(spec, g, 3, exact))
    with open(OUT, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(f"wrote {OUT}: {len(out['updates'])} update sequences, {len(out['peels'])} peels")


if __name__ == "__main__":
    main()
