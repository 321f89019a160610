#!/usr/bin/env python3
"""Per-item beam-search cost vs label size (oracle counters) on a bench workload: does |C_l| predict
an item's V / iterations well enough to schedule long items first?  python scripts/item_cost.py [sift]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from workload import gen, graphs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "sift"
w = gen.make_workload(name, n_queries=10000)
c = w.cfg
go, gi = graphs.build_graphs(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, device=torch.device("cuda"))
o = oracle.Index(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi)
op = "and" if c.query_mode != "single" else "single"
for itopk in (16, 64):
    _, _, ctr = o.search(w.Q, w.q_off, w.q_lab, k=10, itopk=itopk, search_width=2, op=op, counters=True)
    sz = np.diff(w.post_off)
    rec = ctr.reshape(-1, 4)
    rec = rec[rec[:, 1] == oracle.PATH_GRAPH]
    S, V, E = sz[rec[:, 0]], rec[:, 2], rec[:, 3]
    print(f"itopk {itopk}: items {len(S)} corr(log S, V) {np.corrcoef(np.log(S), V)[0, 1]:.3f} "
          f"corr(log S, E) {np.corrcoef(np.log(S), E)[0, 1]:.3f}")
    for lo, hi in [(2000, 10000), (10000, 50000), (50000, 200000), (200000, 10**8)]:
        m = (S >= lo) & (S < hi)
        if m.any():
            print(f"  |C_l| in [{lo}, {hi}): {m.sum():5d} items  V mean {V[m].mean():7.1f}  p99 {np.percentile(V[m], 99):7.1f}"
                  f"  E mean {E[m].mean():5.1f}")
