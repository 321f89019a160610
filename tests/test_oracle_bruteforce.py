"""Oracle vs brute force on tiny inputs, and the invariants the paper fixes."""
import itertools

import numpy as np
import pytest

import oracle
from conftest import small_random_index


def _numpy_filtered_knn(X, point_sets, q, Lq, op, k):
    """Independent brute force: python sets + numpy exact distances (int64 / fp64)."""
    Lq = set(Lq)
    if not Lq:
        return [-1] * k, [np.inf] * k
    if op == "or":
        mask = np.array([bool(s & Lq) for s in point_sets])
    else:
        mask = np.array([Lq <= s for s in point_sets])
    idx = np.flatnonzero(mask)
    if X.dtype == np.uint8:
        d = ((X[idx].astype(np.int64) - q.astype(np.int64)) ** 2).sum(1).astype(np.float64)
    else:
        d = ((X[idx].astype(np.float64) - q.astype(np.float64)) ** 2).sum(1)
    order = np.lexsort((idx, d))[:k]
    ids = idx[order].tolist() + [-1] * (k - len(order))
    ds = d[order].tolist() + [np.inf] * (k - len(order))
    return ids, ds


@pytest.mark.parametrize("dtype", ["f32int", "u8", "f32float"])
@pytest.mark.parametrize("op", ["single", "and", "or"])
def test_exact_knn_vs_numpy_bruteforce(dtype, op):
    cfg, X, off, ids, go, gi = small_random_index(seed=100 + len(op), dtype=dtype)
    ix = oracle.Index(X, off, ids, cfg.threshold_T, cfg.degree_R, go, gi)
    sets = [set() for _ in range(cfg.n_points)]
    for l in range(cfg.n_labels):
        for p in ids[off[l]:off[l + 1]]:
            sets[p].add(l)
    rng = np.random.default_rng(5)
    Q = X[rng.integers(0, cfg.n_points, 40)].copy()
    if dtype != "u8":
        Q = Q + rng.integers(-3, 4, size=Q.shape).astype(np.float32) * (1 if dtype == "f32int" else 1e-3)
    nl = 1 if op == "single" else 2
    ql = rng.integers(0, cfg.n_labels, size=40 * nl).astype(np.int32)
    qo = np.arange(0, 40 * nl + 1, nl, dtype=np.int64)
    got, gd = ix.exact_knn(Q, qo, ql, k=7, op=op)
    for i in range(40):
        e_ids, e_d = _numpy_filtered_knn(X, sets, Q[i], ql[qo[i]:qo[i + 1]].tolist(), op, 7)
        assert got[i].tolist() == e_ids
        np.testing.assert_array_equal(gd[i], np.array(e_d))


@pytest.mark.parametrize("op,mode", [("single", "greedy"), ("and", "greedy"), ("and", "parallel"),
                                     ("or", "greedy")])
def test_exact_mode_equals_definition1(op, mode):
    """Two independent computations agree: the method in exact mode (T = inf: every item scans its
    posting list, then merge) and Definition 1 over all N points with plain membership tests."""
    cfg, X, off, ids, go, gi = small_random_index(seed=200)
    ix = oracle.Index(X, off, ids, cfg.threshold_T, cfg.degree_R, go, gi)
    rng = np.random.default_rng(9)
    n = 60
    nl = 1 if op == "single" else 3
    Q = rng.integers(0, 256, size=(n, cfg.dim)).astype(np.float32)
    ql = rng.integers(0, cfg.n_labels + 2, size=n * nl).astype(np.int32)   # some unknown labels
    qo = np.arange(0, n * nl + 1, nl, dtype=np.int64)
    got, gd = ix.search(Q, qo, ql, k=8, op=op, recall_mode=mode, exact=True)
    gt, gtd = ix.exact_knn(Q, qo, ql, k=8, op=op)
    assert (got == gt).all()
    np.testing.assert_array_equal(gd, gtd)


def test_scan_path_is_exact_and_results_pass_filter(tiny, tiny_oracle):
    """Scan-routed items equal exact kNN; every result carries the query label."""
    w, go, gi = tiny
    ids, d, ctr = tiny_oracle.search(w.Q, w.q_off, w.q_lab, k=10, itopk=32, counters=True)
    gt, gd = tiny_oracle.exact_knn(w.Q, w.q_off, w.q_lab, k=10)
    scan = ctr[:, 0, 1] == oracle.PATH_SCAN
    assert scan.sum() > 100
    assert (ids[scan] == gt[scan]).all() and (d[scan] == gd[scan]).all()
    sets = {l: set(w.post_ids[w.post_off[l]:w.post_off[l + 1]].tolist()) for l in range(w.cfg.n_labels)}
    for i in range(len(ids)):
        l = int(w.q_lab[w.q_off[i]])
        assert all(g in sets[l] for g in ids[i] if g >= 0)


def test_and_or_exactness_invariants():
    """Greedy AND with l* in LS is exact; parallel AND with any LS label is exact; OR over LS
    labels is exact; AND results always satisfy every label."""
    cfg, X, off, ids, go, gi = small_random_index(seed=300, N=400, L=10, T=60)
    ix = oracle.Index(X, off, ids, cfg.threshold_T, cfg.degree_R, go, gi)
    sizes = np.diff(off)
    sets = [set() for _ in range(cfg.n_points)]
    for l in range(cfg.n_labels):
        for p in ids[off[l]:off[l + 1]]:
            sets[p].add(l)
    rng = np.random.default_rng(1)
    pairs = [p for p in itertools.combinations(range(cfg.n_labels), 2)]
    Q = rng.integers(0, 256, size=(len(pairs), cfg.dim)).astype(np.float32)
    ql = np.array(pairs, np.int32).reshape(-1)
    qo = np.arange(0, 2 * len(pairs) + 1, 2, dtype=np.int64)
    gt_and, _ = ix.exact_knn(Q, qo, ql, k=5, op="and")
    gt_or, _ = ix.exact_knn(Q, qo, ql, k=5, op="or")
    g_ids, _ = ix.search(Q, qo, ql, k=5, op="and", recall_mode="greedy", itopk=8)
    p_ids, _ = ix.search(Q, qo, ql, k=5, op="and", recall_mode="parallel", itopk=8)
    o_ids, _ = ix.search(Q, qo, ql, k=5, op="or", itopk=8)
    T = cfg.threshold_T
    n_checked = 0
    for i, (a, b) in enumerate(pairs):
        lstar = a if (sizes[a], a) < (sizes[b], b) else b
        if sizes[lstar] < T:
            assert g_ids[i].tolist() == gt_and[i].tolist(); n_checked += 1
        if min(sizes[a], sizes[b]) < T:
            assert p_ids[i].tolist() == gt_and[i].tolist()
        if max(sizes[a], sizes[b]) < T:
            assert o_ids[i].tolist() == gt_or[i].tolist()
        for res in (g_ids[i], p_ids[i]):
            assert all({a, b} <= sets[g] for g in res if g >= 0)
        assert all({a, b} & sets[g] for g in o_ids[i] if g >= 0)
    assert n_checked > 5


def test_beam_determinism_and_batch_independence(tiny, tiny_oracle):
    """Same (index, query, params) -> same result regardless of batch position / size / threads
    (S:L247, L544); the entry sampler keys on query content (reading c.3)."""
    w, go, gi = tiny
    a, ad = tiny_oracle.search(w.Q, w.q_off, w.q_lab, k=10, itopk=32, nthreads=4)
    perm = np.random.default_rng(0).permutation(len(w.Q))[:300]
    ql = w.q_lab[perm]
    b, bd = tiny_oracle.search(w.Q[perm], np.arange(301, dtype=np.int64), ql, k=10, itopk=32,
                               nthreads=1)
    assert (a[perm] == b).all() and (ad[perm] == bd).all()


def test_mean_recall_nondecreasing_in_itopk(tiny, tiny_oracle):
    """Statistical invariant (reading #32): mean recall over >= 1000 queries is non-decreasing
    over the itopk grid (tolerance 0.002) with n_init and w fixed."""
    w, go, gi = tiny
    gt, _ = tiny_oracle.exact_knn(w.Q, w.q_off, w.q_lab, k=10)
    prev = 0.0
    for itopk in (10, 16, 24, 32, 48, 64, 96, 128):
        ids, _ = tiny_oracle.search(w.Q, w.q_off, w.q_lab, k=10, itopk=itopk, n_init=16)
        r, _ = oracle.recall_at_k(ids, gt)
        assert r >= prev - 0.002
        prev = r
    assert prev > 0.99


def test_zero_label_and_empty_queries(tiny_oracle, tiny):
    w, _, _ = tiny
    Q = w.Q[:3]
    qo = np.array([0, 0, 1, 2], np.int64)             # query 0 has no labels
    ql = np.array([w.cfg.n_labels + 5, 0], np.int32)  # query 1 unknown label
    ids, d = tiny_oracle.search(Q, qo, ql, k=4)
    assert (ids[:2] == -1).all() and np.isinf(d[:2]).all()
    assert (ids[2] >= 0).all()
