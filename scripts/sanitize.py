#!/usr/bin/env python3
"""A small end-to-end run of every product kernel family on tiny inputs, for compute-sanitizer:
   compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python scripts/sanitize.py
batched path (route, AND pre-filter incl. large f3 tiles, tensor-core scan, graph, merge; single / AND / OR;
exact mode),
the per-query path (k_small), label sharding over virtual shards, and the graph builder (k_join, pruning).
The persistent serving kernel is left out: it polls host memory the sanitizer serialises."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2506_00812_b200 as vf  # noqa: E402
from workload import gen, graphs  # noqa: E402

w = gen.make_workload("tiny", n_queries=150)
c = w.cfg
X = gen.gen_vectors(gen.config("tiny", dtype="u8"))
Q = gen.gen_query_vectors(gen.config("tiny", dtype="u8"), n=150)
go, gi = graphs.build_graphs(X, w.post_off, w.post_ids, c.threshold_T, c.degree_R)
ix = vf.Index(X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi)
for mode in ("single", "and2", "or2"):
    qo, ql = (w.q_off, w.q_lab) if mode == "single" else gen.gen_query_labels(c, w.post_off, w.post_ids, n=150, mode=mode)
    op = {"single": "single", "and2": "and", "or2": "or"}[mode]
    for exact in (False, True):
        ix.search(Q, qo, ql, k=10, itopk=32, op=op, exact=exact, search_width=2)
    ix.search(Q[:20], qo[:21], ql[:qo[20]], k=10, itopk=32, op=op)            # per-query path
    if op == "and":
        ix.search(Q, qo, ql, k=10, itopk=32, op=op, recall_mode="parallel", and_scan_threshold=400)
        # f3 routing of every HS l*: large pre-filtered tiles with several survivor pieces
        ix.search(Q, qo, ql, k=10, itopk=32, op=op, and_scan_threshold=10 ** 7)
print("search ok")
sh = vf.Index(X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi, virtual_shards=2)
sh.search(Q, w.q_off, w.q_lab, k=10, itopk=32)
print("shards ok")
g2 = vf.build_graphs(X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, exact_max=2000)
print("builder ok", g2[2])
