#!/usr/bin/env python3
"""Graph-builder workload for profiling (ncu -k regex:k_join): a YFCC-shaped index of --points
points, graphs for every label with >= T points via vf_build_graphs; prints the build report."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--points", type=int, default=2_000_000)
ap.add_argument("--exact-max", type=int, default=0)
a = ap.parse_args()
import paper_2506_00812_b200 as vf  # noqa: E402
from workload import gen  # noqa: E402

cfg = gen.config("yfcc", n_points=a.points)
X = gen.gen_vectors(cfg)
off, ids = gen.gen_postings(cfg)
go, gi, rep = vf.build_graphs(X, off, ids, cfg.threshold_T, cfg.degree_R, exact_max=a.exact_max)
print(rep)
