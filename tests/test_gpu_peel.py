"""GPU parity of the peeling consumers (kcg_update_counts, kcg_peel_exact,
kcg_peel_approx; kcg_peel.cu) against the reference's outputs in
tests/golden/peel_cases.json and the reference's known answers
(proj/tests/test_peeling.cpp).  Every call goes through the C ABI."""
import json
import os

import numpy as np
import pytest

from paper_2002_10047_b200 import gen, kcg
from tests import peelcases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cases():
    return peelcases.load()


def complete(n):
    return gen.from_edges(n, np.array([(i, j) for i in range(n) for j in range(i + 1, n)]))


def oriented(g, strat=kcg.DEGREE, eps=1.0):
    h = kcg.DeviceGraph.from_graph(g)
    h.rank(strat, eps, download=False)
    return h


def test_update_sequences(cases):
    for case in cases["updates"]:
        g = peelcases.graph(case["graph"])
        k = case["k"]
        with oriented(g) as h:
            counts = np.array(case["initial"], np.uint64)
            h.direct(download=False)
            _, pv = h.count(k, per_vertex=True)
            assert pv.tolist() == case["initial"]
            peeled = np.zeros(g.n, np.uint8)
            for st in case["steps"]:
                removed, changed = h.update_counts(k, counts, st["batch"], peeled)
                peeled[st["batch"]] = 1
                assert removed == st["removed"], (case["graph"]["params"], k)
                assert changed.tolist() == st["changed"]
                assert counts.tolist() == st["counts"]


def test_peel_outcomes(cases):
    for case in cases["peels"]:
        g = peelcases.graph(case["graph"])
        with oriented(g, case["strategy"], case["strategy_eps"]) as h:
            out = h.peel_exact(case["k"]) if case["exact"] else \
                h.peel_approx(case["k"], case["eps"])
        peelcases.check_outcome(case, out, "gpu")


def test_known_answers_and_errors():
    g = complete(4)
    with oriented(g) as h:
        counts = np.full(4, 3, np.uint64)
        removed, changed = h.update_counts(3, counts, [0], np.zeros(4, np.uint8))
        assert removed == 3 and changed.tolist() == [1, 2, 3]
        assert counts.tolist() == [3, 1, 1, 1]
        counts = np.full(4, 3, np.uint64)
        removed, changed = h.update_counts(3, counts, [0, 1, 2, 3], np.zeros(4, np.uint8))
        assert removed == 4 and changed.tolist() == []
        pe = np.zeros(4, np.uint8)
        pe[2] = 1
        with pytest.raises(ValueError):
            h.update_counts(3, np.full(4, 3, np.uint64), [1, 2], pe)
        with pytest.raises(ValueError):
            h.update_counts(3, np.full(4, 3, np.uint64), [7], np.zeros(4, np.uint8))
        with pytest.raises(ValueError):
            h.update_counts(1, np.full(4, 3, np.uint64), [0], np.zeros(4, np.uint8))
        # inconsistent counts: a decrement below zero is the reference's
        # std::logic_error (peeling.cpp:174-175)
        with pytest.raises(kcg.KcgLogicError):
            h.update_counts(3, np.zeros(4, np.uint64), [0], np.zeros(4, np.uint8))
        with pytest.raises(ValueError):
            h.peel_exact(1)
        with pytest.raises(ValueError):
            h.peel_approx(3, 0.0)
        with pytest.raises(ValueError):
            h.peel_approx(3, -1.0)
    with oriented(complete(5)) as h:
        out = h.peel_exact(3)
        assert out["total_cliques"] == 10 and out["rounds"] == 1
        assert out["best_density"] == 2.0 and out["best_round"] == 0
        assert out["core"].tolist() == [6] * 5
        assert out["dense_vertices"].tolist() == [0, 1, 2, 3, 4]
    with oriented(gen.from_edges(0, np.zeros((0, 2), np.int64))) as h:
        out = h.peel_exact(3)
        assert out["rounds"] == 0 and out["total_cliques"] == 0


def test_peel_approx_config2_properties():
    """Full-size R-MAT s20: approximate peeling of the 4-clique counts.
    Size-independent checks: the clique total equals kcg_count's, the best
    density is at least the whole graph's, rounds are O(log n) and the
    dense set's own 4-clique density (recounted on the induced subgraph)
    equals the reported best density."""
    g = gen.load_config_graph(2, cache=False)
    spec = gen.CONFIGS[2]
    with oriented(g, spec["strategy"], spec["eps"]) as h:
        h.direct(download=False)
        total, _ = h.count(4)
        out = h.peel_approx(4, 0.5)
    assert out["total_cliques"] == total
    assert out["best_density"] >= total / g.n
    assert out["rounds"] <= 4 * 21 + 2
    dense = out["dense_vertices"]
    keep = np.zeros(g.n, bool)
    keep[dense] = True
    src = np.repeat(np.arange(g.n), np.diff(g.offsets).astype(np.int64))
    sel = keep[src] & keep[g.adj] & (src < g.adj)
    local = np.full(g.n, -1, np.int64)
    local[dense] = np.arange(len(dense))
    sub = gen.from_edges(len(dense), np.stack([local[src[sel]], local[g.adj[sel]]], 1))
    with oriented(sub) as hs:
        hs.direct(download=False)
        t_sub, _ = hs.count(4)
    assert t_sub / len(dense) == out["best_density"]


def test_peel_config_goldens():
    """Config-scale peeling against the reference's outcomes
    (tests/golden/peel_configs.json, tools/make_peel_config_goldens.py)."""
    path = os.path.join(peelcases.ROOT, "tests", "golden", "peel_configs.json")
    gold = json.load(open(path))
    for key, ent in sorted(gold.items()):
        g = gen.load_config_graph(ent["config"], cache=False)
        assert g.digest() == ent["graph_digest"], key
        with oriented(g, ent["strategy"], ent["strategy_eps"]) as h:
            out = h.peel_exact(ent["k"]) if ent["exact"] else h.peel_approx(ent["k"], ent["eps"])
        assert out["rounds"] == ent["rounds"], key
        assert str(out["total_cliques"]) == ent["total_cliques"], key
        assert out["best_round"] == ent["best_round"], key
        assert float(out["best_density"]).hex() == ent["best_density"], key
        assert len(out["dense_vertices"]) == ent["num_dense"], key
        assert f"{gen.digest_u32(out['dense_vertices']):016x}" == ent["dense_digest"], key
        if ent["exact"]:
            assert f"{gen.digest_u64(out['core']):016x}" == ent["core_digest"], key


def test_update_counts_random_states_vs_port(port):
    """Arbitrary peeled sets and (even inconsistent) counts: the device's
    two-sided restricted recount equals the C restatement's recount
    differencing, which is the reference's semantics for any input."""
    rng = np.random.default_rng(77)
    for trial in range(12):
        g = gen.gnp(int(rng.integers(10, 60)), float(rng.uniform(0.2, 0.6)), 900 + trial)
        k = int(rng.integers(2, 6))
        peeled = (rng.random(g.n) < 0.3).astype(np.uint8)
        live = np.flatnonzero(peeled == 0)
        if len(live) == 0:
            continue
        batch = np.sort(rng.choice(live, size=min(len(live), int(rng.integers(1, 6))),
                                   replace=False))
        counts = rng.integers(0, 2000, size=g.n).astype(np.uint64)
        c_gpu, c_port = counts.copy(), counts.copy()
        with oriented(g) as h:
            try:
                r_gpu = h.update_counts(k, c_gpu, batch, peeled)
                err_gpu = None
            except kcg.KcgLogicError:
                r_gpu, err_gpu = None, "logic"
        try:
            r_port = port.update_counts(g, k, c_port, batch, peeled)
            err_port = None
        except Exception:  # noqa: BLE001 - status 4 from the port
            r_port, err_port = None, "logic"
        assert err_gpu == err_port, trial
        if err_gpu is None:
            assert r_gpu[0] == r_port[0] and r_gpu[1].tolist() == r_port[1].tolist(), trial
        assert c_gpu.tolist() == c_port.tolist(), trial


def test_peel_random_graphs_vs_port(port):
    rng = np.random.default_rng(5)
    for trial in range(8):
        g = gen.gnp(int(rng.integers(15, 70)), float(rng.uniform(0.2, 0.5)), 4400 + trial)
        for k in (2, 3, 4):
            with oriented(g, kcg.BARENBOIM_ELKIN, 0.5) as h:
                ex = h.peel_exact(k)
                ap = h.peel_approx(k, 0.3)
            pex = port.peel(g, k, True)
            pap = port.peel(g, k, False, 0.3)
            for a, b in ((ex, pex), (ap, pap)):
                assert a["rounds"] == b["rounds"] and a["best_round"] == b["best_round"]
                assert a["total_cliques"] == b["total_cliques"]
                assert float(a["best_density"]).hex() == float(b["best_density"]).hex()
                assert a["dense_vertices"].tolist() == b["dense_vertices"].tolist()
            assert ex["core"].tolist() == pex["core"].tolist()


def test_update_counts_duplicate_batch_is_a_set():
    """Documented difference: a batch with a repeated vertex
    is treated as the set of its vertices -- the result equals the
    de-duplicated batch's (the reference would charge the repeat twice,
    peeling.cpp:143-174)."""
    g = gen.gnp(40, 0.45, 31)
    k = 4
    with oriented(g) as h:
        base, _ = h.count(k, per_vertex=True)
        _, pv = h.count(k, per_vertex=True)
        peeled = np.zeros(g.n, np.uint8)
        c_set, c_dup = pv.copy(), pv.copy()
        r_set = h.update_counts(k, c_set, [3, 7, 11], peeled)
        r_dup = h.update_counts(k, c_dup, [7, 3, 7, 11, 3], peeled)
    assert base > 0 and r_set[0] > 0
    assert r_set[0] == r_dup[0] and r_set[1].tolist() == r_dup[1].tolist()
    assert c_set.tolist() == c_dup.tolist()
