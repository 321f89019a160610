"""Pins of recall@K (reading #24), workload/metrics.py -- the one definition
bench.py and the oracle tests share. Closed forms written out by hand, plus a plain per-query loop
of the textbook definition on random cases."""
import numpy as np

from workload.metrics import recall_at_k, recall_per_query

INF = np.float32(np.inf)


def test_closed_forms_strict():
    gt = np.arange(10)[None]
    assert recall_at_k(gt, gt)[0] == 1.0
    assert recall_at_k(gt + 100, gt)[0] == 0.0
    half = np.concatenate([np.arange(5), np.arange(100, 105)])[None]
    assert recall_at_k(half, gt)[0] == 0.5
    # order inside the row does not matter
    assert recall_at_k(gt[:, ::-1], gt)[0] == 1.0
    # denominator min(K, |GT|): a filter admitting 2 points, both returned -> 1
    short = np.array([[3, 1] + [-1] * 8])
    assert recall_at_k(short, short)[0] == 1.0
    # ... one of the two returned -> 1/2
    assert recall_at_k(np.array([[3] + [-1] * 9]), short)[0] == 0.5
    # empty GT rows are skipped in the mean: (1 + 0) / 2
    rows = np.stack([np.arange(10), np.arange(10) + 50, np.full(10, -1)])
    gts = np.stack([np.arange(10), np.arange(10), np.full(10, -1)])
    assert recall_at_k(rows, gts)[0] == 0.5
    # -1 in the answer never matches -1 padding in GT
    assert recall_at_k(np.full((1, 10), -1), short)[0] == 0.0


def test_closed_forms_tie_aware():
    # GT = ids 0..9 with distances 0..8, 9 (the K-th distance is 9). The answer swaps GT id 9 for
    # id 77 at distance 9 (a tie at the cut-off) and GT id 8 for id 88 at distance 10.
    gt = np.arange(10)[None]
    gd = np.arange(10, dtype=np.float32)[None]
    ans = np.array([[0, 1, 2, 3, 4, 5, 6, 7, 77, 88]])
    d = np.array([[0, 1, 2, 3, 4, 5, 6, 7, 9, 10]], np.float32)
    s, t = recall_at_k(ans, gt, gd, d)
    assert s == 0.8                     # 8 of 10 strict hits
    assert t == 0.9                     # + id 77 (tie at distance 9); 88 is farther -> no credit
    # the tie-aware score is capped at 1
    ans2 = np.array([[0, 1, 2, 3, 4, 5, 6, 7, 8, 9]])
    s2, t2 = recall_at_k(ans2, gt, gd, np.arange(10, dtype=np.float32)[None])
    assert s2 == 1.0 and t2 == 1.0
    # short GT: |GT| = 3, K-th distance = gd[2]
    gts = np.array([[5, 6, 7] + [-1] * 7])
    gds = np.array([[1, 2, 4] + [INF] * 7], np.float32)
    a3 = np.array([[5, 6, 99] + [-1] * 7])
    d3 = np.array([[1, 2, 4] + [INF] * 7], np.float32)
    s3, t3 = recall_at_k(a3, gts, gds, d3)
    assert abs(s3 - 2 / 3) < 1e-12 and t3 == 1.0


def _loop_reference(ids, gt, d, gd, k):
    """The definition, one query at a time, with Python sets."""
    st, ta = [], []
    for i in range(ids.shape[0]):
        g = [x for x in gt[i][:k] if x >= 0]
        if not g:
            continue
        a = [x for x in ids[i][:k] if x >= 0]
        hits = len(set(a) & set(g))
        kth = gd[i][len(g) - 1]
        extra = sum(1 for t, x in enumerate(ids[i][:k]) if x >= 0 and x not in g and d[i][t] == kth)
        st.append(hits / min(k, len(g)))
        ta.append(min(1.0, (hits + extra) / min(k, len(g))))
    return float(np.mean(st)), float(np.mean(ta))


def test_random_cases_vs_loop():
    rng = np.random.default_rng(7)
    for _ in range(50):
        n, k = 40, 10
        gt = np.stack([rng.choice(30, size=k, replace=False) for _ in range(n)])
        gd = np.sort(rng.integers(0, 6, size=(n, k)).astype(np.float32), axis=1)
        m = rng.integers(0, k + 1, size=n)             # short GT rows
        for i in range(n):
            gt[i, m[i]:] = -1
            gd[i, m[i]:] = INF
        ids = np.stack([rng.choice(30, size=k, replace=False) for _ in range(n)])
        d = rng.integers(0, 7, size=(n, k)).astype(np.float32)
        cut = rng.integers(0, k + 1, size=n)
        for i in range(n):
            ids[i, cut[i]:] = -1
        if not (m > 0).any():
            continue
        s, t = recall_at_k(ids, gt, gd, d, k=k)
        rs, rt = _loop_reference(ids, gt, d, gd, k)
        assert abs(s - rs) < 1e-12 and abs(t - rt) < 1e-12


def test_per_query_valid_mask():
    gt = np.array([[1, 2, -1], [-1, -1, -1]])
    ids = np.array([[2, 9, -1], [4, 5, 6]])
    s, t, v = recall_per_query(ids, gt, k=3)
    assert v.tolist() == [True, False] and t is None and s[0] == 0.5
