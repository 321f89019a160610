"""f1 per-query path (small.cu): batches of <= 64 queries are answered by one
launch with one CTA per query. Its results must equal the oracle's -- and therefore the batched
path's -- under the same bar as tests/test_gpu_parity.py: bit-exact ids, distances and per-item
V / E counters on integer-valued data."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
CH = 64          # kSmallMaxBatch: every chunk below takes the per-query path


@pytest.fixture(scope="module")
def vf():
    import torch
    assert torch.cuda.is_available()
    from paper_2506_00812_b200 import build as B
    B.build()
    import paper_2506_00812_b200 as vf
    return vf


def _variant(tiny, dtype):
    from workload import gen
    w, go, gi = tiny
    if dtype == "f32int":
        return w.X, w.Q
    cfg = gen.config("tiny", dtype=dtype)
    return gen.gen_vectors(cfg), gen.gen_query_vectors(cfg)


def _labels(w, op, n):
    from workload import gen
    if op == "single":
        return w.q_off[:n + 1], w.q_lab[:w.q_off[n]]
    return gen.gen_query_labels(w.cfg, w.post_off, w.post_ids, n=n, mode="and2" if op == "and" else "or2")


def _chunks(n):
    return [(s, min(n, s + CH)) for s in range(0, n, CH)]


def _run_chunks(g, Q, qoff, qlab, **kw):
    n = len(qoff) - 1
    ids = np.empty((n, kw["k"]), np.int32)
    d = np.empty((n, kw["k"]), np.float32)
    recs = []
    for s, e in _chunks(n):
        qo = qoff[s:e + 1] - qoff[s]
        ql = qlab[qoff[s]:qoff[e]]
        ids[s:e], d[s:e] = g.search(Q[s:e], qo, ql, **kw)
        st = g.last_stats()
        assert st["kernel_launches"] == 1, "a small batch must take the one-launch per-query path"
        r = g.last_items().copy()
        r[:, 0] += s
        recs.append(r)
    return ids, d, np.concatenate(recs)


def _items_vs_oracle(recs, octr):
    exp = []
    for i in range(octr.shape[0]):
        for t in range(octr.shape[1]):
            if octr[i, t, 0] >= 0:
                exp.append((i, octr[i, t, 0], octr[i, t, 1], octr[i, t, 2], octr[i, t, 3]))
    got = [tuple(int(x) for x in r[:5]) for r in recs]
    assert len(got) == len(exp)
    bad = [(a, b) for a, b in zip(got, exp) if a != tuple(int(x) for x in b)]
    assert not bad, bad[:5]


@pytest.mark.parametrize("op,mode", [("single", "greedy"), ("and", "greedy"), ("and", "parallel"), ("or", "greedy")])
@pytest.mark.parametrize("dtype", ["f32int", "u8"])
@pytest.mark.parametrize("itopk", [16, 64])
def test_small_batches_bit_exact(vf, tiny, op, mode, dtype, itopk):
    w, go, gi = tiny
    X, Q = _variant(tiny, dtype)
    n = 320
    qoff, qlab = _labels(w, op, n)
    g = vf.Index(X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi)
    o = oracle.Index(X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi)
    ids, d, recs = _run_chunks(g, Q[:n], qoff, qlab, k=10, itopk=itopk, op=op, recall_mode=mode)
    oi, od, octr = o.search(Q[:n], qoff, qlab, k=10, itopk=itopk, op=op, recall_mode=mode, counters=True)
    assert (ids == oi).all()
    assert (d == od.astype(np.float32)).all()
    _items_vs_oracle(recs, octr)
    # and the batched path (one call over all n queries) returns the same
    bi, bd = g.search(Q[:n], qoff, qlab, k=10, itopk=itopk, op=op, recall_mode=mode)
    assert g.last_stats()["kernel_launches"] > 1
    assert (bi == ids).all() and (bd == d).all()


def test_small_batches_generic_float(vf, tiny):
    """Generic fp32 (tiny-float): scan items within 1e-5 relative of the oracle's fp64, graph
    items overlap >= 0.99 (accumulation order differs), as for the batched path."""
    w, go, gi = tiny
    X, Q = _variant(tiny, "f32float")
    n = 256
    g = vf.Index(X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi)
    o = oracle.Index(X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi)
    ids, d, recs = _run_chunks(g, Q[:n], w.q_off[:n + 1], w.q_lab[:w.q_off[n]], k=10, itopk=32)
    oi, od = o.search(Q[:n], w.q_off[:n + 1], w.q_lab[:w.q_off[n]], k=10, itopk=32)
    fin = np.isfinite(od)
    assert np.allclose(d[fin], od[fin], rtol=1e-5, atol=0)
    scan = recs[:, 2] == oracle.PATH_SCAN
    qs = recs[scan, 0]
    assert (ids[qs] == oi[qs]).mean() > 0.99
    overlap = np.mean([np.intersect1d(ids[i], oi[i]).size / 10 for i in range(n)])
    assert overlap >= 0.99


@pytest.mark.parametrize("thr", [0, 400, 2**30])
def test_small_batches_f3_and_f2(vf, tiny, thr):
    """Selectivity-aware AND routing (f3) and the search-time threshold (f2) on the per-query
    path: HS lists scanned by one CTA through M_HS, predicate first."""
    w, go, gi = tiny
    n = 192
    qoff, qlab = _labels(w, "and", n)
    g = vf.Index(w.X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi)
    o = oracle.Index(w.X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi)
    ids, d, _ = _run_chunks(g, w.Q[:n], qoff, qlab, k=10, itopk=32, op="and", and_scan_threshold=thr)
    oi, od = o.search(w.Q[:n], qoff, qlab, k=10, itopk=32, op="and", and_scan_threshold=thr)
    assert (ids == oi).all() and (d == od.astype(np.float32)).all()
    st = 3000 if thr == 400 else (2**31 - 1 if thr else 0)
    ids, d, _ = _run_chunks(g, w.Q[:n], w.q_off[:n + 1], w.q_lab[:w.q_off[n]], k=10, itopk=32, scan_threshold=st)
    oi, od = o.search(w.Q[:n], w.q_off[:n + 1], w.q_lab[:w.q_off[n]], k=10, itopk=32, scan_threshold=st)
    assert (ids == oi).all() and (d == od.astype(np.float32)).all()


def test_small_batch_out_of_range_query_uses_fp32_rows(vf, tiny):
    """u8 row store in front of integer-valued fp32: a query outside [0, 255] is answered from the
    fp32 rows by its own CTA, the others from the u8 rows -- all exact."""
    w, go, gi = tiny
    g = vf.Index(w.X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi)
    o = oracle.Index(w.X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi)
    Q = w.Q[:48].copy()
    Q[3, 0] = 300.0
    Q[7, 1] = -2.0
    a, ad = g.search(Q, w.q_off[:49], w.q_lab[:w.q_off[48]], k=10, itopk=32)
    b, bd = o.search(Q, w.q_off[:49], w.q_lab[:w.q_off[48]], k=10, itopk=32)
    assert (a == b).all() and (ad == bd.astype(np.float32)).all()


def test_small_batch_device_buffers_and_overflow(vf, tiny):
    import torch
    w, go, gi = tiny
    g = vf.Index(w.X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi)
    o = oracle.Index(w.X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi)
    n = 40
    Q, qo, ql = (torch.from_numpy(np.ascontiguousarray(x)).cuda()
                 for x in (w.Q[:n], w.q_off[:n + 1], w.q_lab[:w.q_off[n]]))
    ids = torch.empty((n, 10), dtype=torch.int32, device="cuda")
    d = torch.empty((n, 10), dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    for itopk in (32, 1024):                 # 1024: the visited set spills to the global table
        g.search_into(Q, qo, ql, ids, d, k=10, itopk=itopk, stream=s, n_query_labels=int(w.q_off[n]))
        s.synchronize()
        b, bd = o.search(w.Q[:n], w.q_off[:n + 1], w.q_lab[:w.q_off[n]], k=10, itopk=itopk)
        assert (ids.cpu().numpy() == b).all() and (d.cpu().numpy() == bd.astype(np.float32)).all()


@pytest.mark.parametrize("dtype", ["f32int", "u8"])
def test_serve_persistent_kernel_matches_oracle(vf, tiny, dtype):
    """vf_serve_* (f1): queries published one at a time into the job ring are answered
    by the resident kernel bit-exactly like the oracle; the ring wraps (capacity 16 < queries) and
    many jobs are in flight at once."""
    w, go, gi = tiny
    X, Q = _variant(tiny, dtype)
    g = vf.Index(X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi)
    o = oracle.Index(X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi)
    n = 300
    oi, od = o.search(Q[:n], w.q_off[:n + 1], w.q_lab[:w.q_off[n]], k=10, itopk=32)
    with g.serve(k=10, itopk=32, capacity=16) as sv:
        # one at a time
        for i in range(0, n, 3):
            t = sv.submit(Q[i], w.q_lab[w.q_off[i]:w.q_off[i + 1]])
            ids, d = sv.wait(t)
            assert (ids == oi[i]).all() and (d == od[i].astype(np.float32)).all(), i
        # pipelined: up to 16 in flight
        tickets = {}
        for i in range(n):
            if len(tickets) == 16:
                j = min(tickets)
                ids, d = sv.wait(tickets.pop(j))
                assert (ids == oi[j]).all() and (d == od[j].astype(np.float32)).all(), j
            tickets[i] = sv.submit(Q[i], w.q_lab[w.q_off[i]:w.q_off[i + 1]])
        for j, t in sorted(tickets.items()):
            ids, d = sv.wait(t)
            assert (ids == oi[j]).all() and (d == od[j].astype(np.float32)).all(), j
        assert sv.info()["submitted"] == n // 3 + n


def test_serve_and_queries_f3(vf, tiny):
    w, go, gi = tiny
    n = 120
    qoff, qlab = _labels(w, "and", n)
    g = vf.Index(w.X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi)
    o = oracle.Index(w.X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi)
    for mode, thr in [("greedy", 0), ("parallel", 0), ("greedy", 400)]:
        oi, od = o.search(w.Q[:n], qoff, qlab, k=10, itopk=32, op="and", recall_mode=mode, and_scan_threshold=thr)
        with g.serve(k=10, itopk=32, op="and", recall_mode=mode, and_scan_threshold=thr, capacity=128) as sv:
            ts = [sv.submit(w.Q[i], qlab[qoff[i]:qoff[i + 1]]) for i in range(n)]
            for i, t in enumerate(ts):
                ids, d = sv.wait(t)
                assert (ids == oi[i]).all() and (d == od[i].astype(np.float32)).all(), (mode, thr, i)


def test_serve_rejects_bad_arguments(vf, tiny):
    w, go, gi = tiny
    g = vf.Index(w.X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi)
    with pytest.raises(vf.VfError):
        g.serve(k=64, itopk=64)                       # k > 32 is not served
    with g.serve(k=5, itopk=16, capacity=4) as sv:
        with pytest.raises(vf.VfError):
            sv.submit(w.Q[0], np.arange(17, dtype=np.int32))    # > 16 labels
        with pytest.raises(vf.VfError):
            sv.wait(99)                                # unknown ticket
        t = sv.submit(w.Q[0], w.q_lab[:1])
        ids, _ = sv.wait(t)
        assert ids.shape == (5,)


def test_serve_run_single_batch_mode(vf, tiny):
    """vf_serve_run: a host batch submitted as one job per query (C client loop) equals vf_search."""
    w, go, gi = tiny
    g = vf.Index(w.X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi)
    a, ad = g.search(w.Q, w.q_off, w.q_lab, k=10, itopk=48)
    with g.serve(k=10, itopk=48, capacity=256) as sv:
        b, bd = sv.run(w.Q, w.q_off, w.q_lab, max_in_flight=200)
    assert (a == b).all() and (ad == bd).all()
