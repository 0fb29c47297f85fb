import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def ref():
    """The compiled, unmodified reference (oracle/_ref/libkclique_ref.so)."""
    from tests import reforacle
    try:
        return reforacle.Ref()
    except FileNotFoundError:
        pytest.skip("oracle/_ref/libkclique_ref.so not built (needs /root/reference)")


@pytest.fixture(scope="session")
def port():
    """The C restatement oracle (oracle/_ref/libkcoracle.so)."""
    from tests import reforacle
    return reforacle.Port()


@pytest.fixture(scope="session")
def small_cases():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "small_cases.json")) as f:
        return json.load(f)["cases"]


def load_case_graph(case):
    """Rebuilds a small_cases.json graph and checks its digest."""
    import numpy as np
    from paper_2002_10047_b200 import gen
    kind = case["kind"]
    if kind == "gnp":
        n, p, seed = case["params"]
        g = gen.gnp(n, p, seed)
    elif kind == "rmat":
        s, e, seed, perm = case["params"]
        g = gen.rmat(s, e, seed=seed, permute=bool(perm))
    else:
        ed = np.array(case["graph"]["edges"], dtype=np.int64).reshape(-1, 2)
        g = gen.from_edges(case["graph"]["n"], ed)
    assert g.digest() == case["graph"]["digest"], case["name"]
    return g
