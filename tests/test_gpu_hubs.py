"""Sources with thousands of out-neighbours (identity order, vertex 0 joined
to 2,500 / 4,000 / 4,600 others) against the unmodified reference's totals and
per-vertex digests (tests/golden/hub_cases.json, tools/make_hub_goldens.py):
the tiled k = 4 kernel's top bin, the same bin at its shared-memory limit
(1024- vs 512-thread plan), and the global-memory path above its range."""
import json
import os

import pytest

from paper_2002_10047_b200 import gen, kcg
from tests.hubcases import hub_graph

pytestmark = pytest.mark.gpu

CASES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hub_cases.json")))


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_hub_sources_match_reference(case):
    g = hub_graph(*case["params"])
    assert g.digest() == case["digest"]
    with kcg.DeviceGraph.from_graph(g) as h:
        h.rank(kcg.ORIGINAL, 1.0, download=False)
        _, _, mx = h.direct()
        assert mx == case["max_out"]
        for ks, ent in case["counts"].items():
            total, _ = h.count(int(ks))
            assert str(total) == ent["total"], (case["name"], ks)
            if "pv_digest" in ent:
                t2, pv = h.count(int(ks), per_vertex=True)
                assert t2 == total
                assert f"{gen.digest_u64(pv):016x}" == ent["pv_digest"], (case["name"], ks)
