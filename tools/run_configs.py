#!/usr/bin/env python3
"""Runs the full arb-count pipeline on every BASELINE.json config on the
GPU, checks totals / per-vertex digests against tests/golden, and prints
one JSON line per (config, k) with the device-timed phase split.

    python tools/run_configs.py [--configs 1 2 3 4 5] [--reps 3] [--out FILE]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2002_10047_b200 import gen, kcg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", type=int, nargs="+", default=[1, 2, 3, 4, 5])
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--ks", type=int, nargs="*", default=None)
ap.add_argument("--out", default=None)
a = ap.parse_args()
out = open(a.out, "a") if a.out else None


def emit(d):
    line = json.dumps(d)
    print(line, flush=True)
    if out:
        out.write(line + "\n")
        out.flush()


for cid in a.configs:
    spec = gen.CONFIGS[cid]
    gpath = os.path.join(ROOT, "tests", "golden", f"config{cid}.json")
    gold = json.load(open(gpath)) if os.path.exists(gpath) else {}
    t0 = time.time()
    g = gen.load_config_graph(cid, cache=False)
    tgen = time.time() - t0
    with kcg.DeviceGraph.from_graph(g) as h:
        up = h.timings()["upload_ms"]
        ks = a.ks or spec["ks"]
        for k in ks:
            best = None
            for _ in range(a.reps):
                total, _ = h.pipeline(gen.gpu_strategy(spec), spec["eps"], k)
                t = h.timings()
                step = t["rank_ms"] + t["direct_ms"] + t["count_ms"]
                if best is None or step < best[0]:
                    best = (step, dict(t))
            step, t = best
            want = gold.get("counts", {}).get(str(k), {}).get("total")
            ref_s = gold.get("counts", {}).get(str(k), {}).get("t_count_s")
            emit({"config": cid, "k": k, "n": g.n, "m": g.m, "total": str(total),
                  "golden": want, "ok": (str(total) == want) if want else None,
                  "rank_ms": t["rank_ms"], "direct_ms": t["direct_ms"],
                  "count_ms": t["count_ms"], "step_ms": step,
                  "cliques_per_s": total / (t["count_ms"] / 1e3) if t["count_ms"] else None,
                  "oriented_edges_per_s_e2e": g.m / (step / 1e3),
                  "ref_count_s_8cores": ref_s, "stats": h.count_stats(),
                  "gen_s": tgen, "upload_ms": up})
        for ks_, ent in gold.get("per_vertex", {}).items():
            k = int(ks_)
            total, pv = h.count(k, per_vertex=True)
            t = h.timings()
            emit({"config": cid, "k": k, "per_vertex": True, "total": str(total),
                  "ok": str(total) == ent["total"] and
                  f"{gen.digest_u64(pv):016x}" == ent["digest"],
                  "count_ms": t["count_ms"], "download_ms": t["download_ms"],
                  "sum_ok": int(pv.sum(dtype="uint64")) == (k * total) % (1 << 64)})
        if cid == 5 and "per_vertex" not in gold:
            total, pv = h.count(4, per_vertex=True)
            t = h.timings()
            emit({"config": cid, "k": 4, "per_vertex": True, "total": str(total),
                  "pv_digest": f"{gen.digest_u64(pv):016x}", "count_ms": t["count_ms"],
                  "sum_ok": int(pv.sum(dtype="uint64")) == (4 * total) % (1 << 64)})
    del g
