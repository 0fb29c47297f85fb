"""Multi-GPU sharding of the counting step.

Each rank holds the whole graph, runs ranking and the DAG build (replicas),
then counts only the cliques whose lowest-ranked vertex lies in its own
contiguous, work-balanced range of ranks (`kcg_partition_plan` +
`kcg_count_range`; the reference's edge engine splits the same independent
sources over threads, proj/src/counting.cpp:138-198).  The ranges partition
the cliques, so one all-reduce (sum) of the u64 total -- and of the n u64
per-vertex counts when requested -- gives the single-GPU result.  u64 sums
are carried in int64 tensors: two's-complement addition wraps exactly like
the reference's unchecked u64 counters.
"""
from __future__ import annotations

import numpy as np


def source_work(out_off, out_adj, rank, k: int) -> np.ndarray:
    """Per-source work in rank order, as the device computes it
    (kcg_count.cu source_work_kernel): w(r) = 1 + d + sum_{x in N+(r)}
    (1 + d+(x)), plus d^2 for k >= 5.  Inputs: the id-space DAG (offsets,
    targets) and rank[v]."""
    off = np.asarray(out_off, dtype=np.uint64)
    adj = np.asarray(out_adj, dtype=np.int64)
    d = np.diff(off).astype(np.uint64)
    n = len(d)
    cs = np.zeros(len(adj) + 1, np.uint64)
    np.cumsum(1 + d[adj], dtype=np.uint64, out=cs[1:])
    s = cs[off[1:].astype(np.int64)] - cs[off[:-1].astype(np.int64)]
    w_id = 1 + d + s
    if k >= 5:
        w_id = w_id + d * d
    w = np.empty(n, np.uint64)
    w[np.asarray(rank, dtype=np.int64)] = w_id
    return w


def plan(out_off, out_adj, rank, k: int, nparts: int) -> np.ndarray:
    """Host mirror of kcg_partition_plan: bounds[p] = #{r : excl(r) * P <
    T * p} over the exclusive prefix excl of the per-source work, T its
    total; part p owns ranks [bounds[p], bounds[p + 1])."""
    if nparts < 1:
        raise ValueError("nparts must be positive")
    w = source_work(out_off, out_adj, rank, k)
    n = len(w)
    excl = [0] * n
    acc = 0
    wl = w.tolist()
    for r in range(n):
        excl[r] = acc
        acc += wl[r]
    T = acc
    b = np.zeros(nparts + 1, np.uint32)
    import bisect
    ex = [e * nparts for e in excl]
    for p in range(1, nparts):
        b[p] = bisect.bisect_left(ex, T * p)
    b[nparts] = n
    return b


def allreduce_counts(total: int, per_vertex, device=None, group=None):
    """Sums a rank's (total, per_vertex) over the process group."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([np.uint64(total).view(np.int64)], dtype=torch.int64, device=device)
    dist.all_reduce(t, group=group)
    out_total = int(np.int64(t.item()).view(np.uint64))
    out_pv = None
    if per_vertex is not None:
        pv = torch.from_numpy(np.ascontiguousarray(per_vertex).view(np.int64)).to(device)
        dist.all_reduce(pv, group=group)
        out_pv = pv.cpu().numpy().view(np.uint64)
    return out_total, out_pv
