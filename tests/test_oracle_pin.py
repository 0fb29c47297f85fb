"""Pins the C restatement oracle (oracle/kc_oracle.c) against the compiled
reference library and the reference's own known answers.  CPU only."""
import numpy as np
import pytest

from paper_2002_10047_b200 import gen
from tests.conftest import load_case_graph


def test_mt19937_64_restatement():
    # The C++ standard fixes the 10000th output of a default-seeded
    # mt19937_64 ([rand.predef]); gen.gnp relies on this engine.
    mt = gen._MT64(5489)
    for _ in range(9999):
        mt.next()
    assert mt.next() == 9981545732273789042


def _complete(n):
    return gen.gnp(n, 1.1, 1)


def _path(n):
    return gen.from_edges(n, [(v, v + 1) for v in range(n - 1)])


def _two_clumps():
    e = [(u, v) for u in range(4) for v in range(u + 1, 4)]
    e += [(u, v) for u in range(3, 7) for v in range(u + 1, 7)]
    e.append((0, 7))
    return gen.from_edges(8, e)


def _count(port, g, k, pv=False):
    off, adj = port.direct(g, port.rank_degree(g))
    return port.count(g.n, off, adj, k, want_pv=pv)


def test_port_known_answers(port):
    # proj/tests/test_counting.cpp:30-38
    assert _count(port, _complete(6), 4)[0] == 15
    assert _count(port, _complete(6), 6)[0] == 1
    assert _count(port, _complete(6), 7)[0] == 0
    assert _count(port, _two_clumps(), 3)[0] == 8
    assert _count(port, _path(9), 3)[0] == 0
    with pytest.raises(ValueError):
        _count(port, _complete(3), 1)
    # test_counting.cpp:40-46: k = 2 counts edges
    for seed in range(6):
        g = gen.gnp(25, 0.3, seed)
        assert _count(port, g, 2)[0] == g.m


def test_port_orientation_known_answers(port):
    # proj/tests/test_orientation.cpp:54-59, 130-151, 165-172
    r = port.rank_degree(_path(3))
    assert r[0] < r[1] and r[2] < r[1]
    assert list(port.rank_degree(_complete(5))) == [0, 1, 2, 3, 4]
    r, rounds = port.rank_be(_complete(4), 1.0, 2)
    assert rounds == 1 and list(r) == [0, 1, 2, 3]
    star = gen.from_edges(10, [(0, v) for v in range(1, 10)])
    r, rounds = port.rank_be(star, 1.0, 1)
    assert rounds == 2 and r[0] == 9
    assert port.estimate_arboricity(_path(12), 1.0) == 1
    assert 2 <= port.estimate_arboricity(_complete(5), 1.0) <= 3
    with pytest.raises(ValueError):
        port.rank_be(star, -1.0, 1)
    with pytest.raises(ValueError):
        port.rank_be(star, 1.0, 0)


def test_port_matches_fixture_counts(port, small_cases):
    """Port vs the reference's exhaustive counts stored in small_cases."""
    for case in small_cases[:120]:
        g = load_case_graph(case)
        for ks, ent in case["counts"].items():
            total, pv = _count(port, g, int(ks), pv=True)
            assert str(total) == ent["total"], (case["name"], ks)
            if "pv" in ent:
                assert pv.tolist() == ent["pv"], (case["name"], ks)


@pytest.mark.parametrize("seed", range(0, 60, 3))
def test_port_matches_reference(ref, port, seed):
    n = 5 + seed % 26
    g = gen.gnp(n, [0.2, 0.4, 0.6][seed % 3], seed + 5000)
    rg = ref.graph(g)
    try:
        assert np.array_equal(port.rank_degree(g), ref.rank(rg, n, 0)[0])
        assert np.array_equal(port.rank_kcore(g), ref.rank(rg, n, 2)[0])
        for eps in (0.5, 1.0):
            a = port.estimate_arboricity(g, eps)
            assert a == ref.estimate_arboricity(rg, eps)
            r, rounds = port.rank_be(g, eps, a)
            rr, rrounds, _ = ref.rank(rg, n, 4, eps, a)
            assert np.array_equal(r, rr) and rounds == rrounds
        rank = port.rank_degree(g)
        off, adj = port.direct(g, rank)
        dg, _ = ref.direct(rg, rank)
        roff, radj = ref.dg_csr(dg, n, g.m)
        assert np.array_equal(off, roff) and np.array_equal(adj, radj)
        for k in range(2, 8):
            t, pv = port.count(n, off, adj, k, want_pv=True)
            rt, rpv, _ = ref.count(dg, n, k, want_pv=True)
            assert t == rt and np.array_equal(pv, rpv)
        ref.dg_destroy(dg)
    finally:
        ref.graph_destroy(rg)


def test_port_matches_reference_rmat(ref, port):
    g = gen.rmat(11, 1 << 14, seed=3, permute=True)
    rg = ref.graph(g)
    a = port.estimate_arboricity(g, 0.5)
    assert a == ref.estimate_arboricity(rg, 0.5)
    r, rounds = port.rank_be(g, 0.5, a)
    rr, rrounds, _ = ref.rank(rg, g.n, 4, 0.5, a)
    assert np.array_equal(r, rr) and rounds == rrounds
    off, adj = port.direct(g, r)
    dg, _ = ref.direct(rg, r)
    for k in (3, 4, 5):
        t, pv = port.count(g.n, off, adj, k, want_pv=True)
        rt, rpv, _ = ref.count(dg, g.n, k, want_pv=True)
        assert t == rt and np.array_equal(pv, rpv)
    ref.dg_destroy(dg)
    ref.graph_destroy(rg)
