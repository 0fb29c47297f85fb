#!/usr/bin/env python3
"""Breaks the end-to-end C-ABI step (create -> pipeline -> destroy) into its
host-timed parts (development aid for bench.py's e2e leg)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2002_10047_b200 import gen, kcg  # noqa: E402

g = gen.load_config_graph(2, cache=False)
off_p = torch.from_numpy(g.offsets.view(np.int64)).pin_memory()
adj_p = torch.from_numpy(g.adj.view(np.int32)).pin_memory()
for rep in range(5):
    t0 = time.perf_counter()
    h = kcg.DeviceGraph.from_csr_ptr(g.n, off_p.data_ptr(), adj_p.data_ptr())
    t1 = time.perf_counter()
    tot, _ = h.pipeline(4, 0.5, 4)
    t2 = time.perf_counter()
    tm = h.timings()
    h.close()
    t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.2f} ms (upload_ms {tm['upload_ms']:.2f}) pipeline {1e3*(t2-t1):.2f} ms "
          f"(events: rank {tm['rank_ms']:.2f} direct {tm['direct_ms']:.2f} count {tm['count_ms']:.2f}) "
          f"destroy {1e3*(t3-t2):.2f} ms", flush=True)
