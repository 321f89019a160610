#!/usr/bin/env python3
"""YFCC-shaped diagnostics (GPU box): exact mode vs the CPU oracle on the biggest labels, recall by
query class, and the quality of the fixture graphs' kNN lists. Test tooling, not the product path.

  python scripts/diag_yfcc.py [--config yfcc] [--n-check 24]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="yfcc")
    ap.add_argument("--n-check", type=int, default=24)
    ap.add_argument("--skip-graphs", action="store_true")
    a = ap.parse_args()
    import torch
    import oracle
    import paper_2506_00812_b200 as vf
    from workload import gen, graphs
    dev = torch.device("cuda", 0)
    t0 = time.time()
    w = gen.make_workload(a.config)
    c = w.cfg
    sizes = np.diff(w.post_off)
    print(f"workload {time.time() - t0:.1f}s", flush=True)

    # -- 1. exact mode vs the oracle's Definition-1 scan on single-label queries of the biggest labels
    big = np.argsort(-sizes)[:6]
    rng = np.random.default_rng(0)
    n = a.n_check
    ql = rng.choice(big, size=n).astype(np.int32)
    Q = w.Q[:n]
    qo = np.arange(n + 1, dtype=np.int64)
    empty_go = np.zeros(c.n_labels + 1, np.int64)
    T_inf = int(sizes.max()) + 1          # no HS label: no graphs needed for the exact check
    g = vf.Index(w.X, w.post_off, w.post_ids, T_inf, c.degree_R, empty_go, np.zeros(1, np.int32))
    t0 = time.time()
    ids, d = g.search(Q, qo, ql, k=10, exact=True)
    print(f"gpu exact {n} big-label queries: {time.time() - t0:.2f}s stats={g.last_stats()}", flush=True)
    o = oracle.Index(w.X, w.post_off, w.post_ids, T_inf, c.degree_R)
    t0 = time.time()
    oi, od = o.search(Q, qo, ql, k=10, exact=True)
    print(f"oracle exact: {time.time() - t0:.1f}s", flush=True)
    print("EXACT MODE ids equal:", bool((ids == oi).all()), " dists equal:", bool((d == od.astype(np.float32)).all()),
          flush=True)
    bad = np.flatnonzero((ids != oi).any(1))
    for i in bad[:5]:
        print("  q", i, "label", ql[i], "size", sizes[ql[i]], "gpu", ids[i][:5], d[i][:3], "oracle", oi[i][:5], od[i][:3])
    g.close()
    if a.skip_graphs:
        return

    # -- 2. graph kNN-list quality on the biggest labels (forward half vs exact kNN of sampled nodes)
    t0 = time.time()
    go, gi = graphs.build_graphs(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, device=dev)
    print(f"graphs {time.time() - t0:.1f}s", flush=True)
    for l in list(big[:3]) + [int(np.argmin(np.abs(sizes - 600_000)))] + [int(np.argmin(np.abs(sizes - 20_000)))]:
        ids_l = w.post_ids[w.post_off[l]:w.post_off[l + 1]]
        S = ids_l.size
        Xl = torch.from_numpy(w.X[ids_l]).to(dev).float()
        samp = torch.from_numpy(rng.choice(S, size=min(200, S), replace=False)).to(dev)
        dd = torch.cdist(Xl[samp], Xl) ** 2
        dd[torch.arange(samp.numel(), device=dev), samp] = float("inf")
        ex = torch.topk(dd, 8, largest=False).indices.cpu().numpy()
        rows = gi[go[l] * c.degree_R:go[l + 1] * c.degree_R].reshape(S, c.degree_R)[samp.cpu().numpy()]
        hit = np.mean([np.intersect1d(ex[i], rows[i]).size / 8 for i in range(len(ex))])
        print(f"label {l} size {S}: exact-8NN found in the row: {hit:.3f}", flush=True)

    # -- 3. recall by class on the full mixed batch at a few itopk
    gfull = vf.Index(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi)
    m = 5000
    Qm, qom, qlm = w.Q[:m], w.q_off[:m + 1], w.q_lab[:w.q_off[m]]
    gt, gd = gfull.search(Qm, qom, qlm, k=10, op="and", exact=True)
    nl = np.diff(qom)
    first = qlm[qom[:-1]]
    lstar = np.array([min(qlm[qom[i]:qom[i + 1]], key=lambda l: (sizes[l], l)) for i in range(m)])
    graph_q = sizes[lstar] >= c.threshold_T
    for itopk in (32, 128, 512):
        r, _ = gfull.search(Qm, qom, qlm, k=10, itopk=itopk, op="and")
        rec = np.array([np.intersect1d(r[i][r[i] >= 0], gt[i][gt[i] >= 0]).size / max(1, min(10, (gt[i] >= 0).sum()))
                        for i in range(m)])
        has = (gt >= 0).any(1)
        for name, msk in [("single/graph", (nl == 1) & graph_q), ("single/scan", (nl == 1) & ~graph_q),
                          ("and/graph", (nl == 2) & graph_q), ("and/scan", (nl == 2) & ~graph_q)]:
            mm = msk & has
            print(f"itopk {itopk} {name:13s} n={mm.sum():5d} recall={rec[mm].mean():.4f}", flush=True)
    del first


if __name__ == "__main__":
    main()
