"""GPU parity against the reference's outputs (tests/golden/small_cases.json,
written by tools/make_small_goldens.py from the unmodified reference) and
against the C restatement oracle.  Every call goes through the C ABI."""
import numpy as np
import pytest

from paper_2002_10047_b200 import gen, kcg
from tests.conftest import load_case_graph

pytestmark = pytest.mark.gpu

EXACT_RANKINGS = {"degree", "original", "goodrich_pszona", "barenboim_elkin",
                  "barenboim_elkin_eps05"}


def _dag_digest(off, adj):
    return f"{gen.digest_u64(off):016x}:{gen.digest_u32(adj):016x}"


def _check_case(case):
    g = load_case_graph(case)
    with kcg.DeviceGraph.from_graph(g) as h:
        for name, ent in case.get("rankings", {}).items():
            r, rounds, alpha = h.rank(ent["strategy"], ent["eps"])
            assert f"{gen.digest_u32(r):016x}" == ent["rank_digest"], (case["name"], name)
            if "rank" in ent:
                assert r.tolist() == ent["rank"]
            if ent["strategy"] in (kcg.GOODRICH_PSZONA, kcg.BARENBOIM_ELKIN):
                assert rounds == ent["rounds"], (case["name"], name)
            if "alpha" in ent:
                assert alpha == ent["alpha"]
            off, adj, mx = h.direct()
            assert _dag_digest(off, adj) == ent["dag_digest"], (case["name"], name)
            assert mx == ent["max_out"]
        for block, strat, eps in [("counts", kcg.DEGREE, 1.0),
                                  ("counts_original", kcg.ORIGINAL, 1.0),
                                  ("counts_be05", kcg.BARENBOIM_ELKIN, 0.5)]:
            if block not in case:
                continue
            h.rank(strat, eps, download=False)
            h.direct(download=False)
            for ks, ent in case[block].items():
                k = int(ks)
                total, _ = h.count(k)
                assert str(total) == ent["total"], (case["name"], block, k)
                if "pv_digest" in ent:
                    t2, pv = h.count(k, per_vertex=True)
                    assert t2 == total
                    assert f"{gen.digest_u64(pv):016x}" == ent["pv_digest"], (case["name"], k)
                    if "pv" in ent:
                        assert pv.tolist() == ent["pv"]
                    assert int(pv.sum(dtype=np.uint64)) == (k * total) % (1 << 64)


def test_acceptance_battery(small_cases):
    """acceptance criterion 3's 200 seeded graphs, k = 2..7, five orders."""
    for case in small_cases:
        if case["name"].startswith("accept3"):
            _check_case(case)


@pytest.mark.parametrize("name", ["rmat12", "hub1500", "planted50", "planted36"])
def test_tiered_cases(small_cases, name):
    """CTA tier (rmat12), heavy global-memory tier (hub1500), warp-
    cooperative sets > 32 (planted50), explicit-stack large k (planted36)."""
    case = next(c for c in small_cases if c["name"] == name)
    _check_case(case)



@pytest.mark.parametrize("name", ["rmat12", "hub1500"])
def test_repeated_counts_do_not_flicker(small_cases, name):
    """The staging and credit paths use plain stores, ballots and shared
    atomics under warp- and CTA-level ordering: ten repetitions on the same
    resident DAG must give one total and one per-vertex vector (k = 4 runs
    the tiled kernel on hub1500, k = 5 the shared-memory / global tiers)."""
    case = next(c for c in small_cases if c["name"] == name)
    g = load_case_graph(case)
    with kcg.DeviceGraph.from_graph(g) as h:
        h.rank(kcg.DEGREE, 1.0, download=False)
        h.direct(download=False)
        for k in (4, 5):
            seen = set()
            for _ in range(10):
                t, pv = h.count(k, per_vertex=True)
                t2, _ = h.count(k)
                assert t2 == t
                seen.add((t, gen.digest_u64(pv)))
            assert len(seen) == 1, (name, k, seen)


def test_kcore_is_a_degeneracy_order(small_cases, port):
    for case in small_cases[:60]:
        g = load_case_graph(case)
        with kcg.DeviceGraph.from_graph(g) as h:
            r, rounds, _ = h.rank(kcg.KCORE_PARALLEL)
            assert sorted(r.tolist()) == list(range(g.n))
            _, _, mx = h.direct()
        # degeneracy via the sequential heap order restated in the oracle
        off, _ = port.direct(g, port.rank_kcore(g))
        assert mx == (int(np.diff(off).max()) if g.n else 0)


def test_errors_map_to_invalid_argument():
    g = gen.gnp(12, 0.5, 3)
    with kcg.DeviceGraph.from_graph(g) as h:
        with pytest.raises(ValueError):
            h.count(1)
        with pytest.raises(ValueError):
            h.rank(kcg.BARENBOIM_ELKIN, 0.0)
        with pytest.raises(ValueError):
            h.rank(kcg.GOODRICH_PSZONA, -1.0)
        with pytest.raises(ValueError):
            h.rank(99)
        with pytest.raises(ValueError):
            h.set_ranking([0] * g.n)
        with pytest.raises(ValueError):
            h.set_ranking(list(range(g.n - 1)))
    with pytest.raises(ValueError):
        kcg.rank_barenboim_elkin(g, 1.0, 0)
    # a DAG whose edge points down in rank is rejected
    with pytest.raises(ValueError):
        kcg.DeviceGraph.from_dag([0, 1, 1], [1], [1, 0])


def test_empty_and_edgeless_graphs():
    for g in [gen.from_edges(0, np.zeros((0, 2))), gen.from_edges(7, np.zeros((0, 2)))]:
        with kcg.DeviceGraph.from_graph(g) as h:
            for strat in (kcg.DEGREE, kcg.KCORE, kcg.KCORE_PARALLEL, kcg.BARENBOIM_ELKIN,
                          kcg.GOODRICH_PSZONA):
                r, _, _ = h.rank(strat, 1.0)
                assert sorted(r.tolist()) == list(range(g.n))
            h.direct()
            for k in (2, 3, 5):
                t, pv = h.count(k, per_vertex=True)
                assert t == 0 and not pv.any()


def test_oracle_port_random_sweep(port):
    """Random R-MAT / Chung-Lu graphs, both orders, k = 3..6, vs the port."""
    for seed in range(4):
        for g in (gen.rmat(10, 6000, seed=seed, permute=True),
                  gen.chung_lu(1500, 2.1, 5.0, 10.0, 2.0, 400.0, seed)):
            with kcg.DeviceGraph.from_graph(g) as h:
                for strat in (kcg.DEGREE, kcg.BARENBOIM_ELKIN):
                    rank, _, alpha = h.rank(strat, 0.5)
                    off, adj, _ = h.direct()
                    for k in range(3, 7):
                        total, pv = h.count(k, per_vertex=True)
                        want, want_pv = port.count(g.n, off, adj, k, want_pv=True)
                        assert total == want and np.array_equal(pv, want_pv), (seed, strat, k)


def test_reference_shaped_python_api():
    g = gen.gnp(20, 0.5, 77)
    rank = kcg.make_ranking(g, kcg.OrientConfig(kcg.BARENBOIM_ELKIN, 1.0))
    dg = kcg.direct_by_ranking(g, rank)
    t, pv = kcg.count_per_vertex(dg, 4)
    assert kcg.count_total(dg, 4) == t
    assert int(pv.sum()) == 4 * t


def test_kcore_exact_matches_reference():
    """KCG_KCORE reproduces the reference's sequential (degree, id) heap
    order bit for bit (tests/golden/kcore_cases.json, config 4's golden)."""
    import json
    import os
    from tests import peelcases
    gold = json.load(open(os.path.join(peelcases.ROOT, "tests", "golden", "kcore_cases.json")))
    for c in gold["cases"]:
        if c["kind"] == "gnp":
            g = gen.gnp(*c["params"])
        elif c["kind"] == "rmat":
            s, e, seed, perm = c["params"]
            g = gen.rmat(s, e, seed=seed, permute=bool(perm))
        else:
            g = gen.load_config_graph(c["params"][0], cache=False)
        assert g.digest() == c["digest"]
        with kcg.DeviceGraph.from_graph(g) as h:
            r, _, _ = h.rank(kcg.KCORE)
        if "rank" in c:
            assert r.tolist() == c["rank"], c["params"]
        assert f"{gen.digest_u32(r):016x}" == c["rank_digest"], c["params"]
    g4 = json.load(open(os.path.join(peelcases.ROOT, "tests", "golden", "config4.json")))
    g = gen.load_config_graph(4, cache=False)
    with kcg.DeviceGraph.from_graph(g) as h:
        r, _, _ = h.rank(kcg.KCORE)
    assert f"{gen.digest_u32(r):016x}" == g4["rank_digest"]


def test_concurrent_handles_from_host_threads():
    """SURVEY.md §8(b) threading: one handle per host thread (each with its
    own streams, recycled through the handle pool) gives identical results
    when the calls overlap."""
    import threading
    g = gen.rmat(12, 1 << 15, seed=7, permute=True)
    with kcg.DeviceGraph.from_graph(g) as h:
        want = h.pipeline(kcg.BARENBOIM_ELKIN, 0.5, 4, per_vertex=True)
    results, errors = [], []

    def work():
        try:
            for _ in range(5):
                with kcg.DeviceGraph.from_graph(g) as hh:
                    results.append(hh.pipeline(kcg.BARENBOIM_ELKIN, 0.5, 4, per_vertex=True))
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    threads = [threading.Thread(target=work) for _ in range(6)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    assert len(results) == 30
    for total, pv in results:
        assert total == want[0] and np.array_equal(pv, want[1])
