#!/usr/bin/env python3
"""A/B timing of library switches (environment variables read per search) on one loaded workload.

  python scripts/ab_env.py --config yfcc --itopk 48 --w 2 --and-scan 2000 VF_WARP_SCAN=0 VF_WARP_SCAN=1

Loads the workload, fixture graphs and index once; for each setting: W warm-up searches, K timed
searches (256 MiB L2 flush before each, CUDA events around vf_search), median per-phase device
times (vf_get_last_stats) and the checksum of the results (settings must agree). Test tooling.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("settings", nargs="+")
    ap.add_argument("--config", default="sift")
    ap.add_argument("--itopk", type=int, default=16)
    ap.add_argument("--w", type=int, default=2)
    ap.add_argument("--and-scan", type=int, default=0)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    import torch
    import bench
    import paper_2506_00812_b200 as vf
    dev = torch.device("cuda", 0)
    w, go, gi = bench.make_inputs(a.config, dev)
    c = w.cfg
    ix = vf.Index(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi, device=0)
    ix.set_profiling(True)
    op = "and" if c.query_mode in ("and2", "mix_and") else "single"
    Q, qo, ql = (torch.from_numpy(x).to(dev) for x in (w.Q, w.q_off, w.q_lab))
    n = len(w.Q)
    ids = torch.empty((n, c.k), dtype=torch.int32, device=dev)
    dd = torch.empty((n, c.k), dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device=dev)
    s = torch.cuda.current_stream()
    kw = dict(k=c.k, itopk=a.itopk, search_width=a.w, op=op, and_scan_threshold=a.and_scan, stream=s,
              n_query_labels=int(w.q_off[-1]))
    for setting in a.settings:
        pairs = [kv.split("=") for kv in setting.split(",")]      # NAME=V[,NAME=V...]
        for name, val in pairs:
            os.environ[name] = val
        for _ in range(a.warmup):
            ix.search_into(Q, qo, ql, ids, dd, **kw)
        evs = []
        for _ in range(a.steps):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            ix.search_into(Q, qo, ql, ids, dd, **kw)
            e1.record(s)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        st = ix.last_stats(s)
        ms = float(np.median([e0.elapsed_time(e1) for e0, e1 in evs]))
        chk = int(ids.sum().item())
        print(f"{setting:40s} step {ms:8.3f} ms  QPS {n / ms * 1e3 / 1e6:7.2f}M  route {st['ms_route']:.3f} "
              f"filter {st['ms_filter']:.3f} scan {st['ms_scan']:.3f} graph {st['ms_graph']:.3f}  checksum {chk}",
              flush=True)
        for name, _ in pairs:
            del os.environ[name]


if __name__ == "__main__":
    main()
