#!/usr/bin/env python3
"""Small-batch latency anatomy (BASELINE.json configs[3]): times blocking vf_search calls at batch
1 / 10 / 100 on the SIFT-like index and, under ncu (NVTX range "lat"), lists the kernels one call
launches and their device durations.  python scripts/lat_profile.py [--config sift] [--calls 20]"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2506_00812_b200 as vf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="sift")
ap.add_argument("--calls", type=int, default=200)
ap.add_argument("--itopk", type=int, default=16)
ap.add_argument("--w", type=int, default=2)
args = ap.parse_args()
dev = torch.device("cuda", 0)
w, go, gi = bench.make_inputs(args.config, dev)
c = w.cfg
ix = vf.Index(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi, device=0)
op = "and" if c.query_mode in ("and2", "mix_and") else "single"
st = torch.cuda.current_stream()
for bsz in (1, 10, 100):
    Qd = torch.from_numpy(w.Q[:bsz].copy()).to(dev)
    qod = torch.from_numpy(w.q_off[:bsz + 1].copy()).to(dev)
    qld = torch.from_numpy(w.q_lab[:w.q_off[bsz]].copy()).to(dev)
    oid = torch.empty((bsz, c.k), dtype=torch.int32, device=dev)
    odd = torch.empty((bsz, c.k), dtype=torch.float32, device=dev)
    kw = dict(k=c.k, itopk=args.itopk, search_width=args.w, op=op, stream=st, n_query_labels=int(w.q_off[bsz]))
    for _ in range(20):
        ix.search_into(Qd, qod, qld, oid, odd, **kw)
    torch.cuda.synchronize()
    ts = []
    torch.cuda.nvtx.range_push(f"lat{bsz}")
    for i in range(args.calls):
        t0 = time.perf_counter()
        ix.search_into(Qd, qod, qld, oid, odd, **kw)
        st.synchronize()
        ts.append(time.perf_counter() - t0)
    torch.cuda.nvtx.range_pop()
    # host-side cost alone: enqueue without waiting
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(args.calls):
        ix.search_into(Qd, qod, qld, oid, odd, **kw)
    t_enq = (time.perf_counter() - t0) / args.calls
    torch.cuda.synchronize()
    ix.set_profiling(True)
    for i in range(10):
        ix.search_into(Qd, qod, qld, oid, odd, **kw)
    s = ix.last_stats(st)
    ix.set_profiling(False)
    print(f"batch {bsz}: p50 {1e3 * np.percentile(ts, 50):.3f} ms  enqueue {1e3 * t_enq:.3f} ms/call  "
          f"phases route {s['mean_ms_route']:.3f} scan {s['mean_ms_scan']:.3f} graph {s['mean_ms_graph']:.3f} "
          f"merge {s['mean_ms_merge']:.3f} copy {s['mean_ms_copy']:.3f} total {s['mean_ms_total']:.3f}  "
          f"launches {s['kernel_launches']}", flush=True)
