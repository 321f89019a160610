"""Pins of the CPU oracle against values the paper prints and hand-derived worked examples.

Every test here checks oracle/ against something other than itself: PAPER.md worked examples
(golden fixtures in tests/golden/, each with its citation), closed forms and special cases.
"""
import numpy as np
import pytest

import oracle
from conftest import golden


# ----------------------------------------------------------------------------- predicate
def test_predicate_worked_example_P_L537():
    g = golden("predicate_trace.json")
    ok, tr = oracle.verify(g["point_labels"], g["query_labels"], trace=True)
    assert ok is g["result"]
    q = g["query_labels"]
    assert tr[0, 0] == g["found_index"][str(q[0])]          # smallest label 5 at index 2
    assert tr[-1, 0] == g["found_index"][str(q[-1])]        # largest label 11 at index 5
    lo, hi = g["middle_search_range"][str(q[1])]
    assert (tr[1, 1], tr[1, 2]) == (lo, hi)                 # 9 searched only in [3, 4]
    assert tr[1, 0] == 4


@pytest.mark.parametrize("P,expect", [
    ([1, 3, 5, 7, 9, 11, 13, 15], True),   # query equal to the full label set
    ([2], False), ([0, 1], False), ([15, 16], False), ([1, 15], True), ([7], True), ([], True),
    ([1, 4, 15], False),                   # middle label missing inside the bracket
])
def test_predicate_special_cases(P, expect):
    assert oracle.verify([1, 3, 5, 7, 9, 11, 13, 15], P) is expect


def test_predicate_random_vs_naive_subset():
    """10^4 random (point, query) pairs agree with a naive set-containment check."""
    rng = np.random.default_rng(7)
    for _ in range(10_000):
        pl = np.unique(rng.integers(0, 40, size=rng.integers(0, 12)))
        P = np.unique(rng.integers(0, 40, size=rng.integers(1, 5)))
        if rng.random() < 0.5 and pl.size:
            P = np.unique(rng.choice(pl, size=min(pl.size, rng.integers(1, 4)), replace=False))
        assert oracle.verify(pl, P) == set(P.tolist()).issubset(set(pl.tolist()))


# ----------------------------------------------------------------------------- routing
def _route_index(sizes, T, N=None):
    """Posting lists with the given sizes over disjoint-enough point ranges (no graphs needed)."""
    N = N or (max(sizes) + 10)
    off = np.zeros(len(sizes) + 1, np.int64)
    off[1:] = np.cumsum(sizes)
    ids = np.concatenate([np.arange(s, dtype=np.int32) for s in sizes]) if sizes else np.zeros(0, np.int32)
    X = np.zeros((N, 4), np.float32)
    return oracle.Index(X, off, ids, T, 16)


def test_routing_boundary_P_L334():
    """BFS iff |C_l| < T: |C|=2000 at T=2000 -> graph, 1999 -> scan."""
    ix = _route_index([2000, 1999, 1, 0], T=2000)
    qo = np.arange(5, dtype=np.int64)
    ql = np.array([0, 1, 2, 3], np.int32)
    items, _ = ix.route(qo, ql, op="single")
    path = {int(r[1]): int(r[2]) for r in items}
    assert path == {0: oracle.PATH_GRAPH, 1: oracle.PATH_SCAN, 2: oracle.PATH_SCAN}  # label 3 empty
    items, _ = ix.route(qo, ql, op="single", exact=True)
    assert all(int(r[2]) == oracle.PATH_SCAN for r in items)
    ix1 = _route_index([5, 1], T=1)                       # T = 1 -> everything is HS
    items, _ = ix1.route(np.arange(3, dtype=np.int64), np.array([0, 1], np.int32))
    assert all(int(r[2]) == oracle.PATH_GRAPH for r in items)


def test_and_greedy_list_choice_P_L548_L552():
    g = golden("and_list_choice.json")
    for case in g["cases"]:
        names = list(case["sizes"])
        sizes = [case["sizes"][n] for n in names]
        ix = _route_index(sizes, T=2000)
        qo = np.array([0, len(names)], np.int64)
        ql = np.arange(len(names), dtype=np.int32)[::-1].copy()
        items, pred = ix.route(qo, ql, op="and", recall_mode="greedy")
        assert len(items) == 1
        assert names[int(items[0, 1])] == case["chosen"]
        chosen = case["sizes"][case["chosen"]]
        if "reduction" in case:
            assert 1 - chosen / max(sizes) == pytest.approx(case["reduction"])
        # the predicate holds the remaining labels, sorted
        ps, pl = int(items[0, 3]), int(items[0, 4])
        assert sorted(pred[ps:ps + pl].tolist()) == sorted(set(range(len(names))) - {int(items[0, 1])})
        # parallel policy: one item per label
        items, _ = ix.route(qo, ql, op="and", recall_mode="parallel")
        assert sorted(items[:, 1].tolist()) == list(range(len(names)))


def test_and_greedy_tie_lower_label_and_unknown_labels():
    ix = _route_index([100, 100, 50], T=2000)
    items, _ = ix.route(np.array([0, 2], np.int64), np.array([1, 0], np.int32), op="and")
    assert int(items[0, 1]) == 0                                  # tie -> lower label id (#18)
    items, _ = ix.route(np.array([0, 2], np.int64), np.array([0, 99], np.int32), op="and")
    assert len(items) == 0                                        # unknown label -> empty AND
    items, _ = ix.route(np.array([0, 2], np.int64), np.array([0, 99], np.int32), op="or")
    assert items[:, 1].tolist() == [0]                            # OR skips the unknown branch
    items, _ = ix.route(np.array([0, 3], np.int64), np.array([2, 2, 0], np.int32), op="or")
    assert items[:, 1].tolist() == [0, 2]                         # duplicates removed (#22)
    with pytest.raises(ValueError):
        ix.route(np.array([0, 2], np.int64), np.array([0, 1], np.int32), op="single")


# ----------------------------------------------------------------------------- memory model
def test_memory_model_P_L500():
    g = golden("memory_model.json")
    p = g["params"]
    hs, ls, tot, single, mapping = oracle.memory_model_gib(
        p["N"], p["D"], p["R"], p["R_prime"], p["F"], p["F_HS"], p["F_LS"], p["b"])
    tol = g["tolerance"]
    assert hs == pytest.approx(g["gib"]["hs"], abs=tol)
    assert ls == pytest.approx(g["gib"]["ls"], abs=tol)
    assert tot == pytest.approx(g["gib"]["total"], abs=tol)
    assert single == pytest.approx(g["gib"]["single"], abs=tol)
    assert mapping == pytest.approx(g["gib"]["mapping"], abs=tol)


# ----------------------------------------------------------------------------- beam search
def _appendix_b_index(with_and_label=False):
    g = golden("beam_appendix_b.json")
    pts = np.array(g["points_1d"], np.float32)
    rows = np.array(g["rows"], np.int32)
    S = len(pts)
    X = np.zeros((S, 4), np.float32)
    X[:, 0] = pts
    post = [np.arange(S, dtype=np.int32)]
    if with_and_label:
        # label 1 = the odd points plus 7 far-away points, so |C_1| = 10 > |C_0| = 6 and the
        # greedy AND policy searches label 0 filtering by label 1
        far = np.zeros((7, 4), np.float32)
        far[:, 0] = 1000 + np.arange(7)
        X = np.concatenate([X, far])
        post.append(np.concatenate([np.array([1, 3, 5], np.int32), np.arange(S, S + 7, dtype=np.int32)]))
    off = np.zeros(len(post) + 1, np.int64)
    off[1:] = np.cumsum([len(p) for p in post])
    ids = np.concatenate(post)
    R = rows.shape[1]
    goff = np.zeros(len(post) + 1, np.int64)
    goff[1:] = np.cumsum([len(p) for p in post])
    gids = [rows.reshape(-1)]
    if with_and_label:
        n1 = len(post[1])
        gids.append(np.array([[(j + 1) % n1, (j + 2) % n1] for j in range(n1)], np.int32).reshape(-1))
    gids = np.concatenate(gids)
    T = S
    return g, oracle.Index(X, off, ids, T, R, goff, gids)


def test_beam_appendix_b_trace():
    g, ix = _appendix_b_index()
    q = np.zeros((1, 4), np.float32)
    q[0, 0] = g["query_1d"]
    ids, d, ctr = ix.search(q, np.array([0, 1], np.int64), np.array([0], np.int32), k=g["k"],
                            itopk=g["itopk"], search_width=1, n_init=g["n_init"],
                            max_iterations=g["max_iterations"], forced_entry=g["forced_entry"],
                            counters=True)
    e = g["expected"]
    assert ids[0].tolist() == e["ids"] and d[0].tolist() == e["dists"]
    assert int(ctr[0, 0, 1]) == oracle.PATH_GRAPH
    assert int(ctr[0, 0, 2]) == e["V"] and int(ctr[0, 0, 3]) == e["E"]
    ids1, _ = ix.search(q, np.array([0, 1], np.int64), np.array([0], np.int32), k=1, itopk=2,
                        n_init=1, max_iterations=100, forced_entry=0)
    assert ids1[0].tolist() == e["ids_k1"]


def test_beam_appendix_b_and_variant():
    g, ix = _appendix_b_index(with_and_label=True)
    a = g["and_variant"]
    q = np.zeros((1, 4), np.float32)
    q[0, 0] = g["query_1d"]
    qo, ql = np.array([0, 2], np.int64), np.array([0, 1], np.int32)
    ids, d = ix.search(q, qo, ql, k=a["k"], itopk=a["itopk"], op="and", recall_mode="greedy",
                       n_init=1, max_iterations=100, forced_entry=a["forced_entry"])
    assert ids[0].tolist() == a["expected"]["ids"] and d[0].tolist() == a["expected"]["dists"]
    gt, _ = ix.exact_knn(q, qo, ql, k=1, op="and")
    assert gt[0].tolist() == a["expected"]["exact_and_answer"]


def test_beam_max_iter_zero_is_topk_of_init_sample(tiny, tiny_oracle):
    """max_iter = 0 -> the result is the best k of the n_init sampled entries (c.5)."""
    w, go, gi = tiny
    sizes = np.diff(w.post_off)
    l = int(np.argmax(sizes))
    S = int(sizes[l])
    Q = w.Q[:20]
    qo = np.arange(21, dtype=np.int64)
    ql = np.full(20, l, np.int32)
    n_init = 16
    # max_iterations <= 0 means "auto" in the API; emulate 0 iterations with a graph whose rows
    # are all empty: then no expansion can add a vertex.
    import oracle as O
    empty = np.full_like(gi, -1)
    ix0 = O.Index(w.X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, empty)
    ids, d = ix0.search(Q, qo, ql, k=10, itopk=32, n_init=n_init, seed=123)
    members = w.post_ids[w.post_off[l]:w.post_off[l + 1]]
    for i in range(20):
        qh = O.query_hash(Q[i])
        ent = sorted({O.entry_hash(123, qh, l, t, S) for t in range(n_init)})
        cand = members[ent]
        dd = ((w.X[cand].astype(np.float64) - Q[i].astype(np.float64)) ** 2).sum(1)
        order = np.lexsort((cand, dd))[:10]
        exp_ids = np.full(10, -1)
        exp_ids[:len(order)] = cand[order]
        assert ids[i].tolist() == exp_ids.tolist()


def test_beam_n_init_covers_label_is_exact(tiny, tiny_oracle):
    """n_init >= S -> every vertex is an entry -> the result equals exhaustive top-k."""
    w, go, gi = tiny
    sizes = np.diff(w.post_off)
    hs = np.flatnonzero(sizes >= w.cfg.threshold_T)
    l = int(hs[np.argmin(sizes[hs])])
    Q = w.Q[:30]
    qo = np.arange(31, dtype=np.int64)
    ql = np.full(30, l, np.int32)
    ids, d = tiny_oracle.search(Q, qo, ql, k=10, itopk=16, n_init=int(sizes[l]))
    gt, gd = tiny_oracle.exact_knn(Q, qo, ql, k=10)
    assert (ids == gt).all() and (d == gd).all()


def test_beam_complete_graph_is_exact():
    """R >= S-1 complete graph: the first expansion reaches every vertex -> exact (c.5)."""
    rng = np.random.default_rng(3)
    S, D = 12, 6
    X = rng.integers(0, 256, size=(S, D)).astype(np.float32)
    rows = np.array([[j for j in range(S) if j != i] for i in range(S)], np.int32)
    off = np.array([0, S], np.int64)
    ids = np.arange(S, dtype=np.int32)
    ix = oracle.Index(X, off, ids, 2, S - 1, np.array([0, S], np.int64), rows.reshape(-1))
    Q = rng.integers(0, 256, size=(25, D)).astype(np.float32)
    qo = np.arange(26, dtype=np.int64)
    ql = np.zeros(25, np.int32)
    got, gd = ix.search(Q, qo, ql, k=5, itopk=S, n_init=1)
    gt, gtd = ix.exact_knn(Q, qo, ql, k=5)
    assert (got == gt).all() and (gd == gtd).all()


def test_beam_single_point_label():
    """S = 1 -> that point with its exact distance."""
    X = np.array([[3, 4, 0, 0], [100, 0, 0, 0]], np.float32)
    ix = oracle.Index(X, np.array([0, 1, 2], np.int64), np.array([1, 0], np.int32), 1, 4,
                      np.array([0, 1, 2], np.int64), np.full(8, -1, np.int32))
    q = np.zeros((1, 4), np.float32)
    ids, d = ix.search(q, np.array([0, 1], np.int64), np.array([0], np.int32), k=3, itopk=4)
    assert ids[0].tolist() == [1, -1, -1] and d[0, 0] == 10000.0 and np.isinf(d[0, 1:]).all()


# ----------------------------------------------------------------------------- merge, recall
def test_merge_identity_dedup_idempotent():
    ids = np.array([[4, 7, 9, -1]], np.int32)
    d = np.array([[1.0, 2.0, 2.0, np.inf]])
    oi, od = oracle.merge(ids, d, 4)
    assert oi.tolist() == [4, 7, 9, -1]                           # one list -> identity
    oi2, od2 = oracle.merge([oi, oi], [od, od], 4)
    assert oi2.tolist() == oi.tolist()                            # idempotent, dedup by gid
    a = np.array([[5, 6, -1, -1], [6, 2, 8, -1]], np.int32)
    ad = np.array([[1.0, 3.0, np.inf, np.inf], [3.0, 3.0, 4.0, np.inf]])
    oi, od = oracle.merge(a, ad, 4)
    assert oi.tolist() == [5, 2, 6, 8] and od.tolist() == [1.0, 3.0, 3.0, 4.0]   # tie -> lower id


def test_merge_random_vs_sort_concat_dedup():
    rng = np.random.default_rng(11)
    for _ in range(200):
        n, k = int(rng.integers(1, 5)), int(rng.integers(1, 8))
        pool = rng.permutation(30)[:n * k]
        dist_of = {int(p): float(rng.integers(0, 6)) for p in pool}
        lists, dl = [], []
        for _t in range(n):
            sel = rng.choice(pool, size=k, replace=False)
            m = int(rng.integers(0, k + 1))
            sel = sorted(sel[:m].tolist(), key=lambda g: (dist_of[g], g))
            lists.append(sel + [-1] * (k - m))
            dl.append([dist_of[g] for g in sel] + [np.inf] * (k - m))
        oi, od = oracle.merge(np.array(lists, np.int32), np.array(dl), k)
        uniq = sorted({g for l in lists for g in l if g >= 0}, key=lambda g: (dist_of[g], g))[:k]
        assert oi.tolist() == uniq + [-1] * (k - len(uniq))


def test_recall_closed_forms():
    gt = np.arange(10)[None]
    assert oracle.recall_at_k(gt, gt)[0] == 1.0
    assert oracle.recall_at_k(gt + 100, gt)[0] == 0.0
    half = np.concatenate([np.arange(5), np.arange(100, 105)])[None]
    assert oracle.recall_at_k(half, gt)[0] == 0.5
    short = np.array([[3, 1, -1, -1, -1, -1, -1, -1, -1, -1]])
    assert oracle.recall_at_k(short, short)[0] == 1.0              # denominator min(K, |GT|)


def test_selectivity_aware_and_routing_f3():
    """SURVEY §8(f) f3 (beyond the paper, opt-in): est = |C_l*| * prod |C_o| / N. Hand example:
    N = 10,000, |C_A| = 5,000 (HS at T = 2,000), |C_B| = 6,000 -> l* = A, est = 5000*6000/10000 = 3000."""
    sizes = [5000, 6000]
    off = np.array([0, 5000, 11000], np.int64)
    ids = np.concatenate([np.arange(5000), np.arange(4000, 10000)]).astype(np.int32)
    X = np.zeros((10000, 4), np.float32)
    ix = oracle.Index(X, off, ids, 2000, 16)
    qo, ql = np.array([0, 2], np.int64), np.array([0, 1], np.int32)
    for thr, path in [(0, oracle.PATH_GRAPH), (3000, oracle.PATH_GRAPH), (3001, oracle.PATH_SCAN)]:
        items, _ = ix.route(qo, ql, op="and", and_scan_threshold=thr)
        assert len(items) == 1 and int(items[0, 1]) == 0 and int(items[0, 2]) == path, (thr, items)
    assert sizes[0] < sizes[1]


def test_f3_infinite_threshold_makes_greedy_and_exact(tiny, tiny_oracle):
    """With f3 on for every item, greedy AND scans l*'s list with the predicate: exactly Definition 1."""
    from workload import gen
    w, _, _ = tiny
    qoff, qlab = gen.gen_query_labels(w.cfg, w.post_off, w.post_ids, n=300, mode="and2")
    Q = w.Q[:300]
    ids, d = tiny_oracle.search(Q, qoff, qlab, k=10, op="and", and_scan_threshold=2**30)
    gt, gd = tiny_oracle.exact_knn(Q, qoff, qlab, k=10, op="and")
    assert (ids == gt).all() and (d == gd).all()


def test_scan_threshold_routing_f2():
    """SURVEY §8(f) f2 (the T sweep, P:L339 / P:L766-L768): a search-time threshold T' routes
    |C_l| < max(T, T') to the scan. Hand example at T = 2000: |C_A| = 5,000 is HS; T' = 5,000
    keeps it on the graph (5000 < 5000 is false, P:L334's strict '<'), T' = 5,001 scans it;
    T' below T cannot send the LS label |C_B| = 1,500 to a graph it does not have."""
    off = np.array([0, 5000, 6500], np.int64)
    ids = np.concatenate([np.arange(5000), np.arange(3000, 4500)]).astype(np.int32)
    X = np.zeros((10000, 4), np.float32)
    ix = oracle.Index(X, off, ids, 2000, 16)
    qo, ql = np.array([0, 1, 2], np.int64), np.array([0, 1], np.int32)
    for thr, pa in [(0, oracle.PATH_GRAPH), (1000, oracle.PATH_GRAPH), (5000, oracle.PATH_GRAPH),
                    (5001, oracle.PATH_SCAN), (2**31 - 1, oracle.PATH_SCAN)]:
        items, _ = ix.route(qo, ql, op="single", scan_threshold=thr)
        assert [int(x) for x in items[:, 2]] == [pa, oracle.PATH_SCAN], (thr, items)


def test_f2_infinite_threshold_equals_definition_1(tiny, tiny_oracle):
    """T' = infinity serves every item by the exact scan: results are Definition 1,
    i.e. the scan-only end of the paper's threshold sweep is exact kNN."""
    w, _, _ = tiny
    Q, qoff, qlab = w.Q[:300], w.q_off[:301], w.q_lab[:w.q_off[300]]
    ids, d = tiny_oracle.search(Q, qoff, qlab, k=10, scan_threshold=2**31 - 1)
    gt, gd = tiny_oracle.exact_knn(Q, qoff, qlab, k=10)
    assert (ids == gt).all() and (d == gd).all()


def test_beam_multi_parent_trace():
    """search_width w > 1: parents = the first w UNEXPANDED entries of Top in key order (c.2
    step 2; readings #8/#9). Hand-derived trace in tests/golden/beam_multi_parent.json."""
    g = golden("beam_multi_parent.json")
    pts = np.array(g["points_1d"], np.float32)
    rows = np.array(g["rows"], np.int32)
    S = len(pts)
    X = np.zeros((S, 4), np.float32)
    X[:, 0] = pts
    ix = oracle.Index(X, np.array([0, S], np.int64), np.arange(S, dtype=np.int32), S, rows.shape[1],
                      np.array([0, S], np.int64), rows.reshape(-1))
    q = np.zeros((1, 4), np.float32)
    q[0, 0] = g["query_1d"]
    for w, key in ((2, "expected_w2"), (1, "expected_w1")):
        ids, d, ctr = ix.search(q, np.array([0, 1], np.int64), np.array([0], np.int32), k=g["k"],
                                itopk=g["itopk"], search_width=w, n_init=g["n_init"],
                                max_iterations=g["max_iterations"], forced_entry=g["forced_entry"],
                                counters=True)
        e = g[key]
        assert ids[0].tolist() == e["ids"] and d[0].tolist() == e["dists"], key
        assert int(ctr[0, 0, 2]) == e["V"] and int(ctr[0, 0, 3]) == e["E"], key


# ----------------------------------------------------------------------------- graph builder (f4)
def test_cagra_rows_hand_example():
    """or_cagra_rows on the hand-derived example of tests/golden/cagra_prune.json."""
    g = golden("cagra_prune.json")
    pruned, rows = oracle.cagra_rows(np.array(g["knn"], np.int32), g["R"])
    assert pruned.tolist() == g["pruned"]
    assert rows.tolist() == g["rows"]


def test_cagra_rows_special_cases_and_invariants():
    rng = np.random.default_rng(3)
    # no detours possible: every list points only at nodes whose lists point elsewhere -> pruned =
    # the first R entries (a star: leaves list the centre first, the centre lists the leaves)
    S, K, R = 9, 4, 2
    knn = np.full((S, K), -1, np.int32)
    knn[0] = [1, 2, 3, 4]
    for x in range(1, S):
        knn[x] = [0] + [-1] * (K - 1)
    pruned, rows = oracle.cagra_rows(knn, R)
    assert pruned[0].tolist() == [1, 2]
    assert all(pruned[x].tolist() == [0, -1] for x in range(1, S))
    # K == R keeps every entry (a permutation of the list)
    for _ in range(20):
        S, K = 30, 8
        knn = np.stack([rng.choice(np.delete(np.arange(S), x), size=K, replace=False) for x in range(S)]).astype(np.int32)
        pruned, rows = oracle.cagra_rows(knn, K)
        assert all(sorted(pruned[x]) == sorted(knn[x]) for x in range(S))
    # random lists: pruned is a subset of the list; rows hold no -1 before a valid entry, no
    # duplicate, no self, and only ids of the forward list or of reverse sources
    for _ in range(20):
        S, K, R = 40, 12, 6
        knn = np.stack([rng.choice(np.delete(np.arange(S), x), size=K, replace=False) for x in range(S)]).astype(np.int32)
        pruned, rows = oracle.cagra_rows(knn, R)
        for x in range(S):
            assert set(pruned[x]) <= set(knn[x])
            r = [v for v in rows[x] if v >= 0]
            assert len(r) == len(set(r)) and x not in r
            assert list(rows[x][:len(r)]) == r
            src = {y for y in range(S) if x in pruned[y]}
            assert set(r) <= set(pruned[x]) | src
            assert list(pruned[x][:R // 2]) == r[:R // 2]     # the forward half comes first


def test_label_knn_hand_and_bruteforce():
    """or_label_knn: the App. B 1-D points (hand: ties broken by local id) and a numpy brute force
    (int64 distances, lexsort by (distance, id)) on a random u8 label."""
    pts = np.array([0, 2, 4, 6, 8, 10], np.float32)
    X = np.zeros((6, 4), np.float32)
    X[:, 0] = pts
    o = oracle.Index(X, np.array([0, 6], np.int64), np.arange(6, dtype=np.int32), 10, 2)
    assert o.label_knn(0, 2).tolist() == [[1, 2], [0, 2], [1, 3], [2, 4], [3, 5], [4, 3]]
    assert o.label_knn(0, 6)[0].tolist() == [1, 2, 3, 4, 5, -1]          # S - 1 < K: -1 padded
    rng = np.random.default_rng(5)
    N, D = 300, 24
    X = rng.integers(0, 256, size=(N, D), dtype=np.uint8)
    ids = np.sort(rng.choice(N, size=120, replace=False)).astype(np.int32)
    o = oracle.Index(X, np.array([0, len(ids)], np.int64), ids, 10, 8)
    got = o.label_knn(0, 10)
    Xl = X[ids].astype(np.int64)
    d = ((Xl[:, None, :] - Xl[None, :, :]) ** 2).sum(-1)
    for j in range(len(ids)):
        cand = np.delete(np.arange(len(ids)), j)
        order = np.lexsort((cand, d[j, cand]))
        assert got[j].tolist() == cand[order][:10].tolist()
