"""Input construction on the device (kcg_build.cu):
Graph::from_edges normalisation and the R-MAT generator, checked against the
host generator library (whose normalisation is pinned to the reference's
Graph::from_edges in test_generators.py) and the config graph digests in
tests/golden (written after checking against the reference's own
Graph::from_edges, tools/make_goldens.py)."""
import json
import os

import numpy as np
import pytest

from paper_2002_10047_b200 import gen, kcg

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def same_csr(h, g):
    off, adj = h.csr()
    assert h.n == g.n and h.m == g.m
    assert np.array_equal(off, g.offsets) and np.array_equal(adj, g.adj)


@pytest.mark.parametrize("seed", range(6))
def test_from_edges_matches_host(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 3000))
    cnt = int(rng.integers(0, 20000))
    e = rng.integers(0, n, size=(cnt, 2))
    e = np.concatenate([e, e[: cnt // 5][:, ::-1], np.stack([e[:50, 0], e[:50, 0]], 1)])
    with kcg.DeviceGraph.from_edges(n, e) as h:
        same_csr(h, gen.from_edges(n, e))


def test_from_edges_edge_cases():
    with kcg.DeviceGraph.from_edges(0, np.zeros((0, 2), np.int64)) as h:
        assert h.n == 0 and h.m == 0
    with kcg.DeviceGraph.from_edges(5, [[1, 1], [3, 3]]) as h:
        assert h.m == 0
        off, _ = h.csr()
        assert off.tolist() == [0] * 6
    with kcg.DeviceGraph.from_edges(3, [[2, 0], [0, 1], [1, 0], [0, 2]]) as h:
        off, adj = h.csr()
        assert off.tolist() == [0, 2, 3, 4] and adj.tolist() == [1, 2, 0, 0]
    with pytest.raises(ValueError):
        kcg.DeviceGraph.from_edges(3, [[0, 3]])
    # a device-built graph runs the whole pipeline
    g = gen.gnp(60, 0.3, 11)
    src = np.repeat(np.arange(g.n), np.diff(g.offsets).astype(np.int64))
    with kcg.DeviceGraph.from_edges(g.n, np.stack([src, g.adj], 1)) as h, \
            kcg.DeviceGraph.from_graph(g) as h2:
        assert h.pipeline(kcg.DEGREE, 1.0, 4) == h2.pipeline(kcg.DEGREE, 1.0, 4)


@pytest.mark.parametrize("scale,samples,seed,permute",
                         [(8, 2000, 1, False), (10, 16384, 3, True), (12, 1 << 15, 7, True),
                          (14, 1 << 18, 5, False)])
def test_rmat_matches_host(scale, samples, seed, permute):
    with kcg.DeviceGraph.rmat(scale, samples, seed=seed, permute=permute) as h:
        same_csr(h, gen.rmat(scale, samples, seed=seed, permute=permute))


@pytest.mark.parametrize("cfg", [2, 5])
def test_rmat_config_digests(cfg):
    """Configs 2 and 5 built entirely on the device hash to the goldens."""
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", f"config{cfg}.json")))
    p = gen.CONFIGS[cfg]["rmat"]
    with kcg.DeviceGraph.rmat(p["scale"], p["samples"], seed=p["seed"],
                              permute=p["permute"]) as h:
        assert h.n == gold["n"] and h.m == gold["m"]
        off, adj = h.csr()
        assert f"{gen.digest_u64(off):016x}:{gen.digest_u32(adj):016x}" == gold["graph_digest"]
