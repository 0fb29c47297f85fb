#!/usr/bin/env python3
"""Quick GPU bring-up check: small seeded graphs vs the compiled reference,
then the config graphs vs tests/golden.  Prints one line per check."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2002_10047_b200 import gen, kcg  # noqa: E402
from tests import reforacle  # noqa: E402

R = reforacle.Ref()
print("device", kcg.device_info(), flush=True)
bad = 0
t0 = time.time()
for seed in range(int(os.environ.get("NSEED", "40"))):
    n = 5 + seed % 26
    g = gen.gnp(n, [0.2, 0.4, 0.6][seed % 3], seed + 31000)
    rg = R.graph(g)
    with kcg.DeviceGraph.from_graph(g) as h:
        for strat in [0, 1, 2, 3, 4]:
            r_gpu, rounds_gpu, alpha = h.rank(strat, 1.0)
            r_ref, rounds_ref, _ = R.rank(rg, g.n, strat, 1.0, 0)
            if strat != 2 and not np.array_equal(r_gpu, r_ref):
                print("RANK MISMATCH", seed, strat, r_gpu, r_ref)
                bad += 1
            if strat in (3, 4) and rounds_gpu != rounds_ref:
                print("ROUNDS MISMATCH", seed, strat, rounds_gpu, rounds_ref)
                bad += 1
            off, tgt, mx = h.direct()
            dg, _ = R.direct(rg, r_gpu)
            roff, radj = R.dg_csr(dg, g.n, g.m)
            if not (np.array_equal(off, roff) and np.array_equal(tgt, radj)):
                print("DAG MISMATCH", seed, strat)
                bad += 1
            for k in range(2, 8):
                tot, pv = h.count(k, per_vertex=True)
                et, epv = R.brute_force(rg, g.n, k)
                tt, _ = h.count(k)
                if tot != et or tt != et or not np.array_equal(pv, epv):
                    print("COUNT MISMATCH", seed, strat, k, tot, tt, et, pv, epv)
                    bad += 1
            R.dg_destroy(dg)
    R.graph_destroy(rg)
print(f"small graphs done, {bad} mismatches, {time.time()-t0:.1f}s", flush=True)

gdir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
for cid in [int(c) for c in os.environ.get("CONFIGS", "1 2").split()]:
    path = os.path.join(gdir, f"config{cid}.json")
    if not os.path.exists(path):
        continue
    gold = json.load(open(path))
    spec = gen.CONFIGS[cid]
    t = time.time()
    g = gen.load_config_graph(cid)
    print(f"[{cid}] generated n={g.n} m={g.m} in {time.time()-t:.1f}s digest_ok="
          f"{g.digest() == gold['graph_digest']}", flush=True)
    with kcg.DeviceGraph.from_graph(g) as h:
        r, rounds, alpha = h.rank(gen.gpu_strategy(spec), spec["eps"])
        off, tgt, mx = h.direct()
        print(f"[{cid}] rank ok={gen.digest_u32(r) == int(gold['rank_digest'], 16)} rounds={rounds}"
              f"/{gold['rank_rounds']} alpha={alpha}/{gold.get('alpha_hat')} maxout={mx}/"
              f"{gold['max_out_degree']} times={h.timings()}", flush=True)
        for ks, ent in gold.get("counts", {}).items():
            k = int(ks)
            for rep in range(3):
                tot, _ = h.count(k)
            tm = h.timings()
            print(f"[{cid}] k={k} total={tot} gold={ent['total']} ok={str(tot) == ent['total']} "
                  f"count_ms={tm['count_ms']:.3f} kernel_ms={tm['count_kernel_ms']:.3f} "
                  f"ref_s={ent['t_count_s']:.2f} stats={h.count_stats()}", flush=True)
        for ks, ent in gold.get("per_vertex", {}).items():
            k = int(ks)
            tot, pv = h.count(k, per_vertex=True)
            tm = h.timings()
            print(f"[{cid}] pv k={k} total={tot} ok={str(tot) == ent['total']} "
                  f"digest_ok={gen.digest_u64(pv) == int(ent['digest'], 16)} "
                  f"count_ms={tm['count_ms']:.3f}", flush=True)
