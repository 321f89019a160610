"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

SIFT-like (configs[1]: 1M x 128 integer-valued fp32, 1,000 Zipf labels, the full 10K-query batch
in ONE vf_search, device buffers, the 0.90 / 0.99 operating points) and a YFCC-shaped index at
1M points (configs[2]'s u8 192-d CLR vectors and 200,386-label Zipf model, F = 10.8, a 20K-query
mixed single / AND2 batch, f3 routing off and on): the GPU answers the whole batch;
a seeded sample of queries is answered one by one by the CPU oracle on the same arrays and must
match bit-exactly (ids, distances, per-item V / E). Exact mode (T = infinity) is checked against the
oracle's brute-force Definition 1 on a sample. The full 10M-point YFCC-shaped index (configs[2] at
its size; ~6 min of fixture-graph building) is checked the same way in the `slow` test at the end."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
SAMPLE = 48


@pytest.fixture(scope="module")
def vf():
    import torch
    assert torch.cuda.is_available()
    from paper_2506_00812_b200 import build as B
    B.build()
    import paper_2506_00812_b200 as vf
    return vf


def _build(name, **overrides):
    import torch
    from workload import gen, graphs
    w = gen.make_workload(name, **overrides)
    c = w.cfg
    go, gi = graphs.build_graphs(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, device=torch.device("cuda"))
    return w, go, gi


def _gpu_batch(vf, g, w, **kw):
    import torch
    n, k = len(w.Q), w.cfg.k
    Q, qo, ql = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (w.Q, w.q_off, w.q_lab))
    ids = torch.empty((n, k), dtype=torch.int32, device="cuda")
    d = torch.empty((n, k), dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    g.search_into(Q, qo, ql, ids, d, k=k, stream=s, n_query_labels=int(w.q_off[-1]), **kw)
    s.synchronize()
    _gpu_batch.last_stats = g.last_stats(s)
    return ids.cpu().numpy(), d.cpu().numpy(), g.last_items(s)


def _sample_check(o, w, ids, d, recs, sample, **kw):
    k = w.cfg.k
    by_q = {}
    for r in recs:
        by_q.setdefault(int(r[0]), []).append(tuple(int(x) for x in r[1:5]))   # label, path, V, E
    for i in sample:
        qo = np.array([0, w.q_off[i + 1] - w.q_off[i]], np.int64)
        ql = w.q_lab[w.q_off[i]:w.q_off[i + 1]]
        oi, od, octr = o.search(w.Q[i:i + 1], qo, ql, k=k, counters=True, **kw)
        assert (ids[i] == oi[0]).all() and (d[i] == od[0].astype(np.float32)).all(), i
        exp = [tuple(int(x) for x in octr[0, t]) for t in range(octr.shape[1]) if octr[0, t, 0] >= 0]
        assert by_q.get(i, []) == exp, (i, by_q.get(i), exp)


@pytest.fixture(scope="module")
def sift():
    return _build("sift")


@pytest.mark.parametrize("itopk", [16, 64])
def test_sift_full_batch_sampled_parity(vf, sift, itopk):
    w, go, gi = sift
    c = w.cfg
    g = vf.Index(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi)
    o = oracle.Index(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi)
    ids, d, recs = _gpu_batch(vf, g, w, itopk=itopk, search_width=2)
    assert _gpu_batch.last_stats["kernel_launches"] > 1                # the batched pipeline
    sample = np.random.default_rng(7).choice(len(w.Q), SAMPLE, replace=False)
    _sample_check(o, w, ids, d, recs, sample, itopk=itopk, search_width=2)


def test_sift_full_batch_exact_mode_is_definition1(vf, sift):
    w, go, gi = sift
    c = w.cfg
    g = vf.Index(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi)
    o = oracle.Index(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi)
    ids, d, _ = _gpu_batch(vf, g, w, exact=True)
    sample = np.random.default_rng(8).choice(len(w.Q), 16, replace=False)
    for i in sample:
        qo = np.array([0, w.q_off[i + 1] - w.q_off[i]], np.int64)
        gt, gd = o.exact_knn(w.Q[i:i + 1], qo, w.q_lab[w.q_off[i]:w.q_off[i + 1]], k=c.k)
        assert (ids[i] == gt[0]).all() and (d[i] == gd[0].astype(np.float32)).all(), i


@pytest.fixture(scope="module")
def yfcc1m():
    return _build("yfcc", n_points=1_000_000, n_queries=20_000)


# the bench's operating-point families on the YFCC-shaped mix: paper routing (greedy / parallel),
# f3 at the 0.90 point, and the 0.99 point (itopk 192-384, w = 4: two 32-child batches per
# iteration, 64 entry samples), each in one batched vf_search
@pytest.mark.parametrize("itopk,w_,mode,thr", [(48, 2, "greedy", 0), (48, 2, "greedy", 2000), (32, 2, "parallel", 0),
                                               (192, 2, "greedy", 50000), (384, 4, "greedy", 50000)])
def test_yfcc_shaped_1m_sampled_parity(vf, yfcc1m, itopk, w_, mode, thr):
    w, go, gi = yfcc1m
    c = w.cfg
    g = vf.Index(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi)
    o = oracle.Index(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi)
    kw = dict(itopk=itopk, search_width=w_, op="and", recall_mode=mode, and_scan_threshold=thr)
    ids, d, recs = _gpu_batch(vf, g, w, **kw)
    sample = np.random.default_rng(9 + thr + itopk).choice(len(w.Q), SAMPLE, replace=False)
    _sample_check(o, w, ids, d, recs, sample, **kw)
    g.close()


@pytest.mark.slow
def test_yfcc_10m_sampled_parity(vf):
    """BASELINE.json configs[2] at its full size (10M x 192 u8, 200,386 labels, the 100K mixed
    batch in one vf_search) with fixture graphs (an oracle input never comes from the CUDA path):
    48 sampled queries bit-exact vs the oracle at the bench's 0.90 (f3 1000 / 2000) and 0.99
    operating points (the 0.99 one with scan and graph serialised)."""
    w, go, gi = _build("yfcc")
    c = w.cfg
    g = vf.Index(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi)
    o = oracle.Index(w.X, w.post_off, w.post_ids, c.threshold_T, c.degree_R, go, gi)
    for itopk, w_, thr in ((32, 2, 1000), (48, 2, 2000), (192, 2, 50000)):
        kw = dict(itopk=itopk, search_width=w_, op="and", and_scan_threshold=thr)
        ids, d, recs = _gpu_batch(vf, g, w, **kw)
        sample = np.random.default_rng(31 + itopk).choice(len(w.Q), SAMPLE, replace=False)
        _sample_check(o, w, ids, d, recs, sample, **kw)
