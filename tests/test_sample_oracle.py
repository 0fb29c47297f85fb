"""The colour-sparsification restatement (oracle/kc_oracle.c kco_sparsify)
pinned against the reference's colorful_sparsify outputs
(tests/golden/sample_cases.json, tools/make_sample_goldens.py)."""
import json
import os

from paper_2002_10047_b200 import gen
from tests import peelcases


def test_sparsify_port_matches_reference(port):
    gold = json.load(open(os.path.join(peelcases.ROOT, "tests", "golden", "sample_cases.json")))
    for c in gold["cases"]:
        if c["graph"]["kind"] == "config":
            continue
        g = peelcases.graph(c["graph"])
        off, adj = port.sparsify(g, c["colors"], c["seed"])
        assert f"{gen.digest_u64(off):016x}:{gen.digest_u32(adj):016x}" == c["digest"]
        assert len(adj) // 2 == c["m"]
