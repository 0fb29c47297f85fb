"""World-size-2 gloo test of the multi-GPU host logic: each rank counts its
part (cliques whose lowest-ranked vertex r has r % world == rank), the
parts are all-reduced, and the sum must equal the single-process count.
The per-part count runs through the C restatement oracle here (no GPU);
bench.py --gpus N runs the same split with kcg_count_part over NCCL."""
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
    L.kco_count_part.argtypes = [ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32,
                                 ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint64),
                                 ctypes.c_void_p]
    total = ctypes.c_uint64(0)
    pv = np.zeros(g.n, np.uint64)
    assert L.kco_count_part(g.n, off.ctypes.data, adj.ctypes.data, rnk.ctypes.data, k, rank,
                            world, ctypes.byref(total), pv.ctypes.data) == 0
    t, apv = shard.allreduce_counts(int(total.value), pv)
    if rank == 0:
        want, want_pv = P.count(g.n, off, adj, k, want_pv=True)
        q.put((t, want, bool(np.array_equal(apv, want_pv)), int(total.value)))
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
    got, want, pv_ok, part0 = q.get(timeout=300)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got == want and pv_ok
    assert 0 < part0 < want  # both ranks did real work
