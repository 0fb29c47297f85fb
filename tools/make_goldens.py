#!/usr/bin/env python3
"""Generates tests/golden/config<N>.json by running the UNMODIFIED reference
library (oracle/_ref/libkclique_ref.so, built from /root/reference by
oracle/Makefile) on the canonical config graphs.

Run once, offline, in the build container: the large
configs take minutes to hours on 8 cores.  Results are appended entry by
entry so a partial run is still usable.

    python tools/make_goldens.py --configs 1 2 4 3 5 [--threads 8]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2002_10047_b200 import gen  # noqa: E402
from tests import reforacle  # noqa: E402

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                          "tests", "golden")


def save(path, obj):
    tmp = path + ".tmp"
    with open(tmp, "w") as f:
        json.dump(obj, f, indent=1, sort_keys=True)
    os.replace(tmp, path)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[1, 2, 4, 3, 5])
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--ks", type=int, nargs="*", default=None,
                    help="override the k list (totals only)")
    args = ap.parse_args()
    R = reforacle.Ref()
    if args.threads:
        R.set_threads(args.threads)
    for cid in args.configs:
        spec = gen.CONFIGS[cid]
        path = os.path.join(GOLDEN_DIR, f"config{cid}.json")
        out = json.load(open(path)) if os.path.exists(path) else {}
        t = time.time()
        g = gen.load_config_graph(cid)
        out.update(dict(config=cid, desc=spec["desc"], n=g.n, m=g.m,
                        graph_digest=g.digest(), max_degree=int(g.degrees().max()),
                        threads=R.max_threads()))
        print(f"[{cid}] graph n={g.n} m={g.m} ({time.time()-t:.1f}s)", flush=True)
        t = time.time()
        rg = R.graph(g)
        assert R.graph_digest(rg, g.n) == g.digest(), "generator != Graph::from_edges"
        print(f"[{cid}] reference Graph built, CSR identical ({time.time()-t:.1f}s)", flush=True)
        strat, eps = spec["strategy"], spec["eps"]
        if strat == gen.BARENBOIM_ELKIN:
            alpha = R.estimate_arboricity(rg, eps)
            out["alpha_hat"] = alpha
        rank, rounds, t_rank = R.rank(rg, g.n, strat, eps, 0)
        out.update(rank_strategy=strat, eps=eps, rank_digest=f"{gen.digest_u32(rank):016x}",
                   rank_rounds=rounds, t_rank_s=t_rank)
        dg, t_dir = R.direct(rg, rank)
        off, adj = R.dg_csr(dg, g.n, g.m)
        out.update(dag_digest=f"{gen.digest_u64(off):016x}:{gen.digest_u32(adj):016x}",
                   max_out_degree=int(np.diff(off).max()), t_direct_s=t_dir)
        save(path, out)
        print(f"[{cid}] rank {t_rank:.2f}s direct {t_dir:.2f}s maxout {out['max_out_degree']}",
              flush=True)
        counts = out.setdefault("counts", {})
        ks = args.ks if args.ks is not None else spec["ks"]
        for k in ks:
            if str(k) in counts:
                continue
            total, _, secs = R.count(dg, g.n, k, parallelism=2, want_pv=False)
            counts[str(k)] = dict(total=str(total), t_count_s=secs)
            save(path, out)
            print(f"[{cid}] k={k} total={total} ({secs:.1f}s)", flush=True)
        pvs = out.setdefault("per_vertex", {})
        for k in (spec["pv_ks"] if args.ks is None else []):
            if str(k) in pvs:
                continue
            total, pv, secs = R.count(dg, g.n, k, parallelism=2, want_pv=True)
            pvs[str(k)] = dict(total=str(total), digest=f"{gen.digest_u64(pv):016x}",
                               sum=str(int(pv.sum(dtype=np.uint64))),
                               max=str(int(pv.max())), nonzero=int((pv != 0).sum()),
                               t_count_s=secs)
            save(path, out)
            print(f"[{cid}] pv k={k} total={total} ({secs:.1f}s)", flush=True)
        R.dg_destroy(dg)
        R.graph_destroy(rg)


if __name__ == "__main__":
    main()
