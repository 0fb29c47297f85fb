"""Multi-GPU split on the device: the
work-balanced contiguous source ranges of kcg_partition_plan equal the host
mirror shard.plan, and the parts kcg_count_part(p, P) sum to kcg_count --
totals and per-vertex arrays -- for P in {2, 3, 8} on configs 2 and 4 and
on the hub1500 heavy-tier case.  This is the exact decomposition
bench.py --gpus N all-reduces over NCCL; one GPU runs the parts in turn."""
import numpy as np
import pytest

from paper_2002_10047_b200 import gen, kcg, shard
from tests.conftest import load_case_graph

pytestmark = pytest.mark.gpu


def _check_parts(h, k, per_vertex, parts_list=(2, 3, 8)):
    want, want_pv = h.count(k, per_vertex=per_vertex)
    for P in parts_list:
        tot = 0
        acc = np.zeros(h.n, np.uint64) if per_vertex else None
        b = h.partition_plan(k, P)
        assert b[0] == 0 and b[-1] == h.n and np.all(np.diff(b.astype(np.int64)) >= 0)
        for p in range(P):
            t, pv = h.count_part(k, p, P, per_vertex=per_vertex)
            t2, _ = h.count_range(k, int(b[p]), int(b[p + 1]))
            assert t == t2, (k, P, p)
            tot = (tot + t) % (1 << 64)
            if per_vertex:
                acc += pv
        assert tot == want, (k, P)
        if per_vertex:
            assert np.array_equal(acc, want_pv), (k, P)
    return want


def _plan_matches_host(h, rank, k, P):
    off, adj, _ = h.direct()
    host = shard.plan(off, adj, rank, k, P)
    assert np.array_equal(h.partition_plan(k, P), host), (k, P)


def test_parts_sum_config2():
    g = gen.load_config_graph(2, cache=False)
    spec = gen.CONFIGS[2]
    with kcg.DeviceGraph.from_graph(g) as h:
        rank, _, _ = h.rank(spec["strategy"], spec["eps"])
        h.direct(download=False)
        _plan_matches_host(h, rank, 4, 8)
        _check_parts(h, 4, per_vertex=False)
        _check_parts(h, 4, per_vertex=True, parts_list=(3,))
        _check_parts(h, 5, per_vertex=False, parts_list=(8,))


def test_parts_sum_config4():
    g = gen.load_config_graph(4, cache=False)
    with kcg.DeviceGraph.from_graph(g) as h:
        rank, _, _ = h.rank(gen.gpu_strategy(gen.CONFIGS[4]), 1.0)
        h.direct(download=False)
        _plan_matches_host(h, rank, 6, 3)
        _check_parts(h, 6, per_vertex=True)


def test_parts_sum_hub1500(small_cases):
    case = next(c for c in small_cases if c["name"] == "hub1500")
    g = load_case_graph(case)
    with kcg.DeviceGraph.from_graph(g) as h:
        rank, _, _ = h.rank(kcg.DEGREE)
        h.direct(download=False)
        for k in (3, 4, 5):
            _plan_matches_host(h, rank, k, 8)
            _check_parts(h, k, per_vertex=True)


def test_range_errors():
    g = gen.rmat(8, 1 << 11, seed=1, permute=True)
    with kcg.DeviceGraph.from_graph(g) as h:
        h.rank(kcg.DEGREE, download=False)
        h.direct(download=False)
        with pytest.raises(ValueError):
            h.count_part(4, 2, 2)
        with pytest.raises(ValueError):
            h.count_range(4, 5, 4)
        with pytest.raises(ValueError):
            h.partition_plan(4, 0)
        assert h.count_range(4, 0, 0)[0] == 0
