#!/usr/bin/env python3
"""Cycle breakdown of the tensor-core scan (diagnostics build, -DVF_TC_PROF): builds the library
with the counters enabled, runs a few searches of a workload and prints the per-role TCPROF lines
of CTAs 0-1 (producer / MMA / two epilogue warps). Test tooling, not the product path.

  VF_NVCC_EXTRA=-DVF_TC_PROF python scripts/tc_prof.py [--config sift] [--itopk 16]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="sift")
    ap.add_argument("--itopk", type=int, default=16)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--and-scan", type=int, default=0)
    a = ap.parse_args()
    from paper_2506_00812_b200 import build as B
    B.build(force=True)
    import torch
    import paper_2506_00812_b200 as vf
    sys.path.insert(0, ROOT)
    import bench
    w, go, gi = bench.make_inputs(a.config, torch.device("cuda", 0))
    c = w.cfg
    ix = vf.Index(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi)
    op = "and" if c.query_mode in ("and2", "mix_and") else "single"
    for _ in range(a.reps):
        ix.search(w.Q, w.q_off, w.q_lab, k=c.k, itopk=a.itopk, search_width=2, op=op, and_scan_threshold=a.and_scan)
        torch.cuda.synchronize()
        print("----", ix.last_stats(), flush=True)


if __name__ == "__main__":
    main()
