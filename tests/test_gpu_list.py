"""GPU clique listing (kcg_list.cu, kcg_list_cliques) against the C
restatement's counts and exhaustive enumeration: every clique once, rows in
ascending rank, batches split by the source-masked counter."""
import itertools

import numpy as np
import pytest

from paper_2002_10047_b200 import gen, kcg

pytestmark = pytest.mark.gpu


def brute(g, k):
    adj = [set(g.adj[g.offsets[v]:g.offsets[v + 1]].tolist()) for v in range(g.n)]
    out = set()
    for c in itertools.combinations(range(g.n), k):
        if all(c[j] in adj[c[i]] for i in range(k) for j in range(i + 1, k)):
            out.add(c)
    return out


@pytest.mark.parametrize("seed", range(4))
def test_list_matches_exhaustive(seed):
    g = gen.gnp(18, 0.6, seed + 300)
    with kcg.DeviceGraph.from_graph(g) as h:
        r, _, _ = h.rank(kcg.DEGREE)
        h.direct(download=False)
        for k in (2, 3, 4, 5, 6):
            total, cl = h.list_cliques(k)
            want = brute(g, k)
            assert total == len(want) == len(cl)
            assert set(tuple(sorted(row)) for row in cl.tolist()) == want
            assert np.all(np.diff(r[cl], axis=1) > 0) if len(cl) else True


def test_list_batches_and_counts(port):
    g = gen.rmat(11, 1 << 14, seed=3, permute=True)
    with kcg.DeviceGraph.from_graph(g) as h:
        h.rank(kcg.BARENBOIM_ELKIN, 0.5, download=False)
        off, adj, _ = h.direct()
        for k in (3, 4, 5):
            want, _ = port.count(g.n, off, adj, k)
            total, cl = h.list_cliques(k, batch=max(1, want // 7))
            assert total == want == len(cl)
            rows = np.sort(cl, axis=1)
            assert len(np.unique(rows, axis=0)) == want
            # every pair of a listed clique is an edge
            src = np.repeat(np.arange(g.n), np.diff(g.offsets).astype(np.int64))
            edges = set(zip(src.tolist(), g.adj.tolist()))
            for row in rows[:: max(1, len(rows) // 500)].tolist():
                assert all((row[i], row[j]) in edges
                           for i in range(k) for j in range(i + 1, k))
    with kcg.DeviceGraph.from_graph(g) as h:
        h.rank(kcg.DEGREE, download=False)
        with pytest.raises(ValueError):
            h.list_cliques(1)
