import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: longer CPU test")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def tiny():
    """BASELINE.json configs[0] (fp32-int variant) with its fixture graphs."""
    from workload import gen, graphs
    w = gen.make_workload("tiny")
    c = w.cfg
    go, gi = graphs.build_graphs(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R)
    return w, go, gi


@pytest.fixture(scope="session")
def tiny_oracle(tiny):
    import oracle
    w, go, gi = tiny
    return oracle.Index(w.X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi)


def small_random_index(seed, N=300, D=8, L=12, F=2.5, T=40, R=8, dtype="f32int"):
    """A small random index for brute-force checks (labels via the Zipf generator)."""
    from workload import gen, graphs
    cfg = gen.config("tiny", n_points=N, dim=D, n_labels=L, mean_labels=F, threshold_T=T,
                     degree_R=R, dtype=dtype)
    X = gen.gen_vectors(cfg, seed=seed)
    off, ids = gen.gen_postings(cfg, seed=seed + 1)
    go, gi = graphs.build_graphs(X, off, ids, T, R)
    return cfg, X, off, ids, go, gi
