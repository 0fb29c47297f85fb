"""Shared loader for tests/golden/peel_cases.json (written from the
unmodified reference by tools/make_peel_goldens.py)."""
import json
import os

import numpy as np

from paper_2002_10047_b200 import gen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load():
    with open(os.path.join(ROOT, "tests", "golden", "peel_cases.json")) as f:
        return json.load(f)


def graph(spec):
    kind, p = spec["kind"], spec["params"]
    if kind == "gnp":
        g = gen.gnp(p[0], p[1], p[2])
    elif kind == "rmat":
        g = gen.rmat(p[0], p[1], seed=p[2], permute=bool(p[3]))
    elif kind == "config":
        g = gen.load_config_graph(p[0])
    else:
        g = gen.from_edges(spec["n"], np.array(spec["edges"], np.int64).reshape(-1, 2))
    assert g.digest() == spec["digest"], spec
    return g


def check_outcome(case, out, where=""):
    """Compares a peel outcome dict with a golden entry."""
    tag = (where, case["graph"]["kind"], case["graph"].get("params"), case["k"],
           case["exact"])
    assert out["rounds"] == case["rounds"], tag
    assert str(out["total_cliques"]) == case["total_cliques"], tag
    assert out["best_round"] == case["best_round"], tag
    assert float(out["best_density"]).hex() == case["best_density"], tag
    dense = np.asarray(out["dense_vertices"], np.uint32)
    assert len(dense) == case["num_dense"], tag
    assert f"{gen.digest_u32(dense):016x}" == case["dense_digest"], tag
    if "dense_vertices" in case:
        assert dense.tolist() == case["dense_vertices"], tag
    if case["exact"]:
        core = np.asarray(out["core"], np.uint64)
        assert f"{gen.digest_u64(core):016x}" == case["core_digest"], tag
        if "core" in case:
            assert core.tolist() == case["core"], tag
