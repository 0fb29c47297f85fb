#!/usr/bin/env python3
"""OPS(k) for config/k pairs with the instrumented CPU
recursion tools/kc_ops.c (built here with gcc -O3 -fopenmp), cross-checked
against the golden totals, and the resulting k >= 5 issue-roofline
fraction of the B200 counts in profiles/r01c_configs.jsonl:

    T_roof = OPS / P_int,  P_int = SMs * 128 lanes * max SM clock
    frac   = T_roof / t_count

    python tools/ops_count.py --pairs 3:5 2:5 [--out FILE]
"""
import argparse
import ctypes
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2002_10047_b200 import gen  # noqa: E402
from tests import reforacle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--pairs", nargs="+", default=["3:5"])
ap.add_argument("--out", default=None)
a = ap.parse_args()
so = os.path.join(ROOT, "tools", "_build", "libkcops.so")
os.makedirs(os.path.dirname(so), exist_ok=True)
subprocess.run(["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-o", so,
                os.path.join(ROOT, "tools", "kc_ops.c")], check=True)
L = ctypes.CDLL(so)
vp = ctypes.c_void_p
L.kc_ops.argtypes = [ctypes.c_uint32, vp, vp, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64),
                     ctypes.POINTER(ctypes.c_uint64)]
P = reforacle.Port()
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"sm_max_mhz": 1965.0}
p_int = 148 * 128 * peaks["sm_max_mhz"] * 1e6
gpu = {}
cfgs = os.path.join(ROOT, "profiles", "r01c_configs.jsonl")
if os.path.exists(cfgs):
    for line in open(cfgs):
        d = json.loads(line)
        if not d.get("per_vertex"):
            gpu[(d["config"], d["k"])] = d["count_ms"]
dags = {}
for pair in a.pairs:
    cid, k = map(int, pair.split(":"))
    spec = gen.CONFIGS[cid]
    if cid not in dags:
        g = gen.load_config_graph(cid, cache=False)
        # the counted DAG is the same up to vertex names for any ranking of
        # the config; use the reference's own strategy through the port
        if spec["strategy"] == gen.DEGREE:
            r = P.rank_degree(g)
        elif spec["strategy"] == gen.BARENBOIM_ELKIN:
            r, _ = P.rank_be(g, spec["eps"], P.estimate_arboricity(g, spec["eps"]))
        else:
            r = P.rank_kcore(g)
        off, adj = P.direct(g, r)
        dags[cid] = (g.n, np.ascontiguousarray(off), np.ascontiguousarray(adj))
    n, off, adj = dags[cid]
    ops, tot = ctypes.c_uint64(0), ctypes.c_uint64(0)
    t0 = time.perf_counter()
    L.kc_ops(n, off.ctypes.data, adj.ctypes.data, k, ctypes.byref(ops), ctypes.byref(tot))
    secs = time.perf_counter() - t0
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", f"config{cid}.json")))
    rec = {"config": cid, "k": k, "ops": int(ops.value), "total": str(tot.value),
           "total_matches_golden": str(tot.value) == gold["counts"][str(k)]["total"],
           "cpu_s": secs, "threads": os.cpu_count(), "p_int_ops_per_s": p_int}
    if (cid, k) in gpu:
        t_roof = ops.value / p_int
        rec.update(t_roof_ms=t_roof * 1e3, gpu_count_ms=gpu[(cid, k)],
                   issue_roofline_frac=t_roof * 1e3 / gpu[(cid, k)])
    line = json.dumps(rec)
    print(line, flush=True)
    if a.out:
        with open(a.out, "a") as f:
            f.write(line + "\n")
