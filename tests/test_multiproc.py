"""World-size-2 gloo test of the multi-GPU host logic: every rank computes
the product's partition plan (shard.plan, the host mirror of
kcg_partition_plan: work-balanced contiguous ranges of source ranks),
counts the cliques whose lowest-ranked vertex lies in its own range, the
parts are all-reduced (shard.allreduce_counts), and the sum must equal the
single-process count.  The per-range count is the C restatement oracle
here (no GPU); bench.py --gpus N runs the same plan with kcg_count_range
over NCCL, and tests/test_gpu_shard.py checks the device plan against
shard.plan."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2002_10047_b200 import gen


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, k, q):
    import ctypes

    import torch.distributed as dist

    from paper_2002_10047_b200 import shard
    from tests import reforacle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P = reforacle.Port()
    g = gen.rmat(11, 1 << 14, seed=21, permute=True)
    rnk = P.rank_degree(g)
    off, adj = P.direct(g, rnk)
    L = P.L
    L.kco_count_range.argtypes = [ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32,
                                  ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint64),
                                  ctypes.c_void_p]
    bounds = shard.plan(off, adj, rnk, k, world)
    total = ctypes.c_uint64(0)
    pv = np.zeros(g.n, np.uint64)
    assert L.kco_count_range(g.n, off.ctypes.data, adj.ctypes.data, rnk.ctypes.data, k,
                             int(bounds[rank]), int(bounds[rank + 1]), ctypes.byref(total),
                             pv.ctypes.data) == 0
    t, apv = shard.allreduce_counts(int(total.value), pv)
    if rank == 0:
        want, want_pv = P.count(g.n, off, adj, k, want_pv=True)
        q.put((t, want, bool(np.array_equal(apv, want_pv)), int(total.value),
               [int(x) for x in bounds]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("k", [3, 4, 5])
def test_two_rank_partition_sums_to_single_count(k):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, k, q)) for r in range(2)]
    for p in ps:
        p.start()
    got, want, pv_ok, part0, bounds = q.get(timeout=300)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got == want and pv_ok
    assert 0 < part0 < want  # both ranks did real work
    assert bounds[0] == 0 and 0 < bounds[1] < bounds[2]


def test_plan_balances_work_and_covers_all_sources():
    """shard.plan: contiguous, monotone ranges covering [0, n) whose work
    shares differ by at most one source's work."""
    from paper_2002_10047_b200 import shard
    from tests import reforacle

    P = reforacle.Port()
    g = gen.rmat(12, 1 << 15, seed=5, permute=True)
    rnk = P.rank_degree(g)
    off, adj = P.direct(g, rnk)
    for k in (4, 5):
        w = shard.source_work(off, adj, rnk, k).astype(np.int64)
        for parts in (1, 2, 3, 8):
            b = shard.plan(off, adj, rnk, k, parts)
            assert b[0] == 0 and b[-1] == g.n and np.all(np.diff(b.astype(np.int64)) >= 0)
            loads = [int(w[b[p]:b[p + 1]].sum()) for p in range(parts)]
            assert sum(loads) == int(w.sum())
            assert max(loads) - min(loads) <= 2 * int(w.max())


def test_range_oracle_matches_part_oracle_sum():
    """The range restatement partitions the cliques like the modulo one."""
    import ctypes

    from tests import reforacle

    P = reforacle.Port()
    g = gen.rmat(10, 1 << 13, seed=3, permute=True)
    rnk = P.rank_degree(g)
    off, adj = P.direct(g, rnk)
    L = P.L
    L.kco_count_range.argtypes = [ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32,
                                  ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint64),
                                  ctypes.c_void_p]
    for k in (3, 4, 5):
        want, want_pv = P.count(g.n, off, adj, k, want_pv=True)
        cuts = [0, g.n // 3, g.n // 2, g.n]
        tot, acc = 0, np.zeros(g.n, np.uint64)
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            t = ctypes.c_uint64(0)
            pv = np.zeros(g.n, np.uint64)
            assert L.kco_count_range(g.n, off.ctypes.data, adj.ctypes.data, rnk.ctypes.data, k,
                                     lo, hi, ctypes.byref(t), pv.ctypes.data) == 0
            tot += t.value
            acc += pv
        assert tot == want and np.array_equal(acc, want_pv)
