#!/usr/bin/env python3
"""Writes tests/golden/hub_cases.json: one vertex with a very large
out-neighbourhood under the identity order (the sources the tiled k = 4
kernel and the global-memory tiers take), counted by the UNMODIFIED reference
(oracle/_ref/libkclique_ref.so).  Run in the build container:
    python tools/make_hub_goldens.py
The graph of a case is rebuilt from its parameters by tests/test_gpu_hubs.py
(gen.rmat + numpy's PCG64 stream) and checked against the stored digest."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2002_10047_b200 import gen  # noqa: E402
from tests import reforacle  # noqa: E402
from tests.hubcases import hub_graph  # noqa: E402


def main():
    R = reforacle.Ref()
    R.set_threads(8)
    cases = []
    # (fan, ks, per-vertex ks): 2500 -> tiled (2047, 4095] bin; 4000 -> the same
    # bin near its shared-memory limit; 4600 -> above the tiled kernel's range
    for fan, ks, pvks in [(2500, [3, 4, 5], [4]), (4000, [4], [4]), (4600, [4], [4])]:
        params = [13, 1 << 17, 100 + fan, fan]
        g = hub_graph(*params)
        rg = R.graph(g)
        r, _, _ = R.rank(rg, g.n, gen.ORIGINAL, 1.0, 0)
        dg, _ = R.direct(rg, r)
        off, _ = R.dg_csr(dg, g.n, g.m)
        ent = {"name": f"hub{fan}", "params": params, "n": g.n, "m": g.m, "digest": g.digest(),
               "max_out": int(np.diff(off).max()), "counts": {}}
        for k in ks:
            total, pv, _ = R.count(dg, g.n, k, want_pv=k in pvks)
            c = {"total": str(total)}
            if k in pvks:
                c["pv_digest"] = f"{gen.digest_u64(pv):016x}"
            ent["counts"][str(k)] = c
        R.dg_destroy(dg)
        R.graph_destroy(rg)
        cases.append(ent)
        print(ent["name"], ent["max_out"], ent["counts"], flush=True)
    with open(os.path.join(ROOT, "tests", "golden", "hub_cases.json"), "w") as f:
        json.dump(cases, f, indent=1)


if __name__ == "__main__":
    main()
