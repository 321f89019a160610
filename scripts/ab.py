#!/usr/bin/env python3
"""A/B timing of several builds of libvecflow on one loaded workload (GPU box).

  python scripts/ab.py --config sift --itopk 16 --w 2 lib_a.so lib_b.so ...

Loads the workload and fixture graphs once, then for each library: build the index, W warm-up
searches, K timed searches (256 MiB L2 flush before each, CUDA events around vf_search), and
prints the median per-phase device times from vf_get_last_stats.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--config", default="sift")
    ap.add_argument("--itopk", type=int, default=16)
    ap.add_argument("--w", type=int, default=2)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--exact", action="store_true")
    a = ap.parse_args()
    import torch
    import paper_2506_00812_b200 as vf
    from workload import gen, graphs
    dev = torch.device("cuda", 0)
    w = gen.make_workload(a.config)
    c = w.cfg
    go, gi = graphs.build_graphs(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, device=dev)
    op = "and" if c.query_mode in ("and2", "mix_and") else "single"
    Q = torch.from_numpy(w.Q).to(dev)
    qo = torch.from_numpy(w.q_off).to(dev)
    ql = torch.from_numpy(w.q_lab).to(dev)
    n = len(w.Q)
    ids = torch.empty((n, c.k), dtype=torch.int32, device=dev)
    dd = torch.empty((n, c.k), dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device=dev)
    s = torch.cuda.current_stream()
    ref = None
    for path in a.libs:
        vf._lib = None
        vf.LIB_PATH = os.path.abspath(path)
        ix = vf.Index(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi, device=0)
        ix.set_profiling(True)
        kw = dict(k=c.k, itopk=a.itopk, search_width=a.w, op=op, exact=a.exact, stream=s)
        for _ in range(a.warmup):
            ix.search_into(Q, qo, ql, ids, dd, **kw)
        st = []
        for _ in range(a.steps):
            flush.fill_(1.0)
            ix.search_into(Q, qo, ql, ids, dd, **kw)
            st.append(ix.last_stats(s))
        torch.cuda.synchronize()
        out = ids.cpu().numpy()
        same = "ref" if ref is None else ("same results" if (out == ref).all() else "RESULTS DIFFER")
        ref = out if ref is None else ref
        med = {p: float(np.median([x[f"ms_{p}"] for x in st])) for p in ("route", "scan", "graph", "merge", "total")}
        print(f"{os.path.basename(path):28s} " + " ".join(f"{p}={v:.4f}" for p, v in med.items()) +
              f"  QPS={n / med['total'] * 1e3 / 1e6:.2f}M  [{same}]", flush=True)
        ix.close()


if __name__ == "__main__":
    main()
