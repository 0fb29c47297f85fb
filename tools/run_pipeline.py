#!/usr/bin/env python3
"""The whole config pipeline on one B200 with nothing on the host but the
parameters: R-MAT samples generated and normalised on the device
(kcg_graph_rmat) -> ranking -> DAG -> per-vertex k-clique counts ->
approximate k-clique densest-subgraph peeling.  Prints one JSON line per
config with the device-timed phases and the checks against tests/golden.

    python tools/run_pipeline.py [--configs 2 5] [--eps 0.5] [--no-peel]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2002_10047_b200 import gen, kcg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", type=int, nargs="+", default=[2, 5])
ap.add_argument("--eps", type=float, default=0.5)
ap.add_argument("--no-peel", action="store_true")
ap.add_argument("--out", default=None)
a = ap.parse_args()


def sync_time(fn):
    t0 = time.perf_counter()
    r = fn()
    return r, (time.perf_counter() - t0) * 1e3


for cid in a.configs:
    spec = gen.CONFIGS[cid]
    p = spec["rmat"]
    k = spec["ks"][0]
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", f"config{cid}.json")))
    h, build_wall = sync_time(lambda: kcg.DeviceGraph.rmat(p["scale"], p["samples"],
                                                           seed=p["seed"],
                                                           permute=p["permute"]))
    rec = {"config": cid, "k": k, "n": h.n, "m": h.m, "build_ms": h.timings()["upload_ms"],
           "build_wall_ms": build_wall}
    off, adj = h.csr()
    rec["graph_digest_ok"] = f"{gen.digest_u64(off):016x}:{gen.digest_u32(adj):016x}" == \
        gold["graph_digest"]
    del off, adj
    h.rank(gen.gpu_strategy(spec), spec["eps"], download=False)
    rec["rank_ms"] = h.timings()["rank_ms"]
    h.direct(download=False)
    rec["direct_ms"] = h.timings()["direct_ms"]
    total, pv = h.count(k, per_vertex=True)
    t = h.timings()
    rec.update(total=str(total), count_pv_ms=t["count_ms"], pv_download_ms=t["download_ms"],
               total_ok=str(total) == gold["counts"][str(k)]["total"],
               pv_sum_ok=int(pv.sum(dtype=np.uint64)) == (k * total) % (1 << 64),
               pv_digest=f"{gen.digest_u64(pv):016x}")
    gpv = gold.get("per_vertex", {}).get(str(k))
    if gpv:
        rec["pv_digest_ok"] = rec["pv_digest"] == gpv["digest"]
    if not a.no_peel:
        out, ms = sync_time(lambda: h.peel_approx(k, a.eps))
        rec.update(peel_ms=ms, peel_rounds=out["rounds"], peel_best_round=out["best_round"],
                   peel_best_density=out["best_density"], peel_dense=len(out["dense_vertices"]),
                   peel_total_ok=out["total_cliques"] == total)
        pg = os.path.join(ROOT, "tests", "golden", "peel_configs.json")
        if os.path.exists(pg):
            ent = json.load(open(pg)).get(f"config{cid}_k{k}_approx")
            if ent and ent["eps"] == a.eps:
                rec["peel_golden_ok"] = (
                    out["rounds"] == ent["rounds"] and out["best_round"] == ent["best_round"]
                    and out["best_density"].hex() == ent["best_density"]
                    and f"{gen.digest_u32(out['dense_vertices']):016x}" == ent["dense_digest"])
                rec["peel_ref_seconds"] = ent["ref_seconds"]
    rec["device_gb"] = h.device_bytes() / 1e9
    h.close()
    line = json.dumps(rec)
    print(line, flush=True)
    if a.out:
        with open(a.out, "a") as f:
            f.write(line + "\n")
