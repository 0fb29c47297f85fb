"""Graphs of tests/golden/hub_cases.json (shared by tools/make_hub_goldens.py,
which asks the reference for the counts, and tests/test_gpu_hubs.py)."""
import numpy as np

from paper_2002_10047_b200 import gen


def hub_graph(scale, samples, seed, fan):
    """R-MAT base graph plus vertex 0 joined to `fan` random other vertices."""
    base = gen.rmat(scale, samples, seed=seed, permute=True)
    off = np.asarray(base.offsets, dtype=np.int64)
    adj = np.asarray(base.adj, dtype=np.int64)
    src = np.repeat(np.arange(base.n, dtype=np.int64), np.diff(off))
    keep = src < adj
    rng = np.random.default_rng(seed)
    hub = rng.choice(np.arange(1, base.n), fan, replace=False).astype(np.int64)
    e = np.concatenate([np.stack([src[keep], adj[keep]], 1),
                        np.stack([np.zeros(fan, np.int64), hub], 1)])
    return gen.from_edges(base.n, e)
