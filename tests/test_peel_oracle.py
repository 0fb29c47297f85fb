"""The peeling restatement in oracle/kc_oracle.c (kco_update_counts,
kco_peel) pinned against the reference's outputs (peel_cases.json) and the
reference's own known answers (proj/tests/test_peeling.cpp)."""
import numpy as np
import pytest

from paper_2002_10047_b200 import gen
from tests import peelcases


@pytest.fixture(scope="module")
def cases():
    return peelcases.load()


def complete(n):
    return gen.from_edges(n, np.array([(i, j) for i in range(n) for j in range(i + 1, n)]))


def test_update_sequences_match_reference(port, cases):
    for case in cases["updates"]:
        g = peelcases.graph(case["graph"])
        k = case["k"]
        counts = np.array(case["initial"], np.uint64)
        peeled = np.zeros(g.n, np.uint8)
        for st in case["steps"]:
            removed, changed = port.update_counts(g, k, counts, st["batch"], peeled)
            peeled[st["batch"]] = 1
            assert removed == st["removed"]
            assert changed.tolist() == st["changed"]
            assert counts.tolist() == st["counts"]


def test_peel_outcomes_match_reference(port, cases):
    for case in cases["peels"]:
        if case["graph"]["n"] > 1100 or case["graph"]["kind"] == "config":
            continue
        g = peelcases.graph(case["graph"])
        out = port.peel(g, case["k"], case["exact"], case["eps"])
        peelcases.check_outcome(case, out, "port")


def test_known_answers(port):
    # test_peeling.cpp:62-76: one vertex of K_4 tears three triangles out
    g = complete(4)
    counts = np.full(4, 3, np.uint64)
    removed, changed = port.update_counts(g, 3, counts, [0], np.zeros(4, np.uint8))
    assert removed == 3 and changed.tolist() == [1, 2, 3] and counts.tolist() == [3, 1, 1, 1]
    # :78-88 whole-graph batch counts every triangle once
    counts = np.full(4, 3, np.uint64)
    removed, changed = port.update_counts(g, 3, counts, [0, 1, 2, 3], np.zeros(4, np.uint8))
    assert removed == 4 and changed.tolist() == []
    # :90-99 a peeled batch vertex is rejected
    pe = np.zeros(4, np.uint8)
    pe[2] = 1
    with pytest.raises(ValueError):
        port.update_counts(g, 3, np.full(4, 3, np.uint64), [1, 2], pe)
    # :150-159 K_5 peels in one round at density 2
    out = port.peel(complete(5), 3, True)
    assert out["total_cliques"] == 10 and out["rounds"] == 1 and out["best_density"] == 2.0
    assert out["core"].tolist() == [6] * 5 and out["dense_vertices"].tolist() == [0, 1, 2, 3, 4]
    # :194-207 approximate peeling of K_5 and a path
    out = port.peel(complete(5), 3, False, 0.5)
    assert out["rounds"] == 1 and out["best_density"] == 2.0
    path = gen.from_edges(8, np.array([[i, i + 1] for i in range(7)]))
    out = port.peel(path, 3, False, 0.5)
    assert out["total_cliques"] == 0 and out["rounds"] == 1 and out["best_density"] == 0.0
