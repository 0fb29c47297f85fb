"""GPU colour sparsification and approximate counting (kcg_sample.cu,
kcg_colorful_sparsify / kcg_approx_count) against the reference's outputs
(tests/golden/sample_cases.json).  Every call goes through the C ABI."""
import json
import os

import pytest

from paper_2002_10047_b200 import gen, kcg
from tests import peelcases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gold():
    return json.load(open(os.path.join(peelcases.ROOT, "tests", "golden", "sample_cases.json")))


def test_sparsify_and_approx_count(gold):
    for c in gold["cases"]:
        g = peelcases.graph(c["graph"])
        with kcg.DeviceGraph.from_graph(g) as h:
            with h.colorful_sparsify(c["colors"], c["seed"]) as s:
                off, adj = s.csr()
                assert f"{gen.digest_u64(off):016x}:{gen.digest_u32(adj):016x}" == c["digest"]
                assert s.m == c["m"]
            for key, want in c["approx"].items():
                k, strat, eps = key.split(":")
                e = h.approx_count(int(k), c["colors"], c["seed"], int(strat), float(eps))
                assert str(e["sub_count"]) == want["sub_count"], (c["graph"]["params"], key)
                assert float(e["p"]).hex() == want["p"]
                assert float(e["estimate"]).hex() == want["estimate"]


def test_sparsify_errors():
    g = gen.gnp(10, 0.5, 1)
    with kcg.DeviceGraph.from_graph(g) as h:
        with pytest.raises(ValueError):
            h.colorful_sparsify(0, 1)
        with pytest.raises(ValueError):
            h.approx_count(1, 2, 1)
        with pytest.raises(ValueError):
            h.approx_count(3, 0, 1)
