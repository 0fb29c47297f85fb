"""Multi-GPU sharding of the counting step.

Each rank holds the whole graph, runs ranking and the DAG build (replicas),
then counts only the cliques whose lowest-ranked vertex r satisfies
r % world == rank (`kcg_count_part`).  The parts partition the cliques, so
one all-reduce (sum) of the u64 total — and of the n u64 per-vertex counts
when requested — produces the single-GPU result.  u64 sums are carried in
int64 tensors: two's-complement addition wraps exactly like the reference's
unchecked u64 counters.
"""
from __future__ import annotations

import numpy as np


def part_of(rank: int, world: int) -> tuple[int, int]:
    return rank, world


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
