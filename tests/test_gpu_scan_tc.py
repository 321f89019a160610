"""The tensor-core scan (scan_tc.cu: tcgen05.mma kind::i8 for u8, kind::tf32 for integer-valued
fp32; TMA tensor loads) vs the oracle.

u8 distances are exact int32 on both sides (||x||^2 + ||q||^2 - 2 q.x on the GPU, sum of squared
differences in the oracle), so ids and distances must be bit-identical (BASELINE.json north_star:
"bit-exact for int8"). The cases cover every swizzle width the kernel picks (row bytes a multiple
of 128 / 64 / 32, and K padding when it is none of these), 1..64 queries per segment (MMA N 16..64),
k on both sides of the register-list limit (32), multi-stage and multi-tile labels, HS rows
gathered per row (exact mode and f3 routing) and the AND predicate inside the epilogue.
"""
import numpy as np
import pytest

import oracle
from conftest import small_random_index

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vf():
    import torch
    assert torch.cuda.is_available()
    from paper_2506_00812_b200 import build as B
    B.build()
    import paper_2506_00812_b200 as vf
    return vf


def _u8_scan_index(dim, N=4000, L=9, seed=5):
    """u8 vectors, L labels of ragged sizes (some > 4 stages of 128 rows), every label LS."""
    rng = np.random.default_rng(seed)
    X = rng.integers(0, 256, size=(N, dim), dtype=np.uint8)
    sizes = [1, 37, 128, 129, 255, 600, 1024, 1500, N]
    sizes = sizes[:L]
    ids = [np.sort(rng.choice(N, size=s, replace=False)).astype(np.int32) for s in sizes]
    off = np.zeros(L + 1, np.int64)
    off[1:] = np.cumsum([len(i) for i in ids])
    return X, off, np.concatenate(ids)


def _queries(dim, n, labels, seed):
    rng = np.random.default_rng(seed)
    Q = rng.integers(0, 256, size=(n, dim), dtype=np.uint8)
    qoff = np.arange(n + 1, dtype=np.int64)
    qlab = rng.choice(labels, size=n).astype(np.int32)
    return Q, qoff, qlab


@pytest.mark.parametrize("dim", [16, 32, 48, 128, 192, 200])
def test_u8_scan_all_swizzle_widths(vf, dim):
    X, off, ids = _u8_scan_index(dim)
    T = 1 << 30                                     # every label LS: the result is Definition 1
    g = vf.Index(X, off, ids, T, 8)
    o = oracle.Index(X, off, ids, T, 8)
    Q, qoff, qlab = _queries(dim, 700, np.arange(len(off) - 1), seed=dim)
    for k in (1, 10, 40):
        a, ad = g.search(Q, qoff, qlab, k=k, itopk=max(k, 16))
        e, ed = o.exact_knn(Q, qoff, qlab, k=k)
        assert (a == e).all(), (dim, k)
        assert (ad == ed.astype(np.float32)).all(), (dim, k)


def test_u8_scan_full_query_groups(vf):
    """Many queries on one label: segments of up to 64 queries (MMA N = 64)."""
    dim = 192
    X, off, ids = _u8_scan_index(dim)
    g = vf.Index(X, off, ids, 1 << 30, 8)
    o = oracle.Index(X, off, ids, 1 << 30, 8)
    Q, qoff, _ = _queries(dim, 300, [0], seed=3)
    qlab = np.array([5, 7] * 150, np.int32)          # 150 queries on each of two labels
    a, ad = g.search(Q, qoff, qlab, k=10, itopk=16)
    e, ed = o.exact_knn(Q, qoff, qlab, k=10)
    assert (a == e).all() and (ad == ed.astype(np.float32)).all()
    st = g.last_stats()
    assert st["n_segments"] >= 6                     # 150 queries -> >= 3 segments per label


@pytest.mark.parametrize("op", ["single", "and", "or"])
def test_u8_exact_mode_hs_gathers(vf, op):
    """exact=1 streams HS labels too, rows gathered from X through M_HS (TMA tile::gather4)."""
    from workload import gen
    cfg, X, off, ids, go, gi = small_random_index(seed=11, N=3000, D=192, L=10, F=2.0, T=300, R=8,
                                                  dtype="u8")
    assert (np.diff(off) >= 300).any()
    g = vf.Index(X, off, ids, cfg.threshold_T, cfg.degree_R, go, gi)
    o = oracle.Index(X, off, ids, cfg.threshold_T, cfg.degree_R, go, gi)
    Q = gen.gen_query_vectors(cfg, n=400)
    if op == "single":
        qoff = np.arange(401, dtype=np.int64)
        qlab = np.random.default_rng(1).integers(0, cfg.n_labels, size=400).astype(np.int32)
    else:
        qoff, qlab = gen.gen_query_labels(cfg, off, ids, n=400, mode=op + "2")
    a, ad = g.search(Q, qoff, qlab, k=10, op=op, exact=True)
    e, ed = o.exact_knn(Q, qoff, qlab, k=10, op=op)
    assert (a == e).all() and (ad == ed.astype(np.float32)).all()


@pytest.mark.parametrize("thr", [60, 2**30])
def test_u8_f3_routing(vf, thr):
    from workload import gen
    cfg, X, off, ids, go, gi = small_random_index(seed=12, N=3000, D=64, L=10, F=2.5, T=300, R=8,
                                                  dtype="u8")
    g = vf.Index(X, off, ids, cfg.threshold_T, cfg.degree_R, go, gi)
    o = oracle.Index(X, off, ids, cfg.threshold_T, cfg.degree_R, go, gi)
    Q = gen.gen_query_vectors(cfg, n=400)
    qoff, qlab = gen.gen_query_labels(cfg, off, ids, n=400, mode="and2")
    a, ad = g.search(Q, qoff, qlab, k=10, itopk=32, op="and", and_scan_threshold=thr)
    e, ed = o.search(Q, qoff, qlab, k=10, itopk=32, op="and", and_scan_threshold=thr)
    assert (a == e).all() and (ad == ed.astype(np.float32)).all()


def test_u8_multi_tile_exact(vf):
    """Labels spanning several 4096-row tiles in exact mode: partial lists merged in-kernel."""
    dim = 96
    rng = np.random.default_rng(9)
    N = 20000
    X = rng.integers(0, 256, size=(N, dim), dtype=np.uint8)
    off = np.array([0, N, N + 9000], np.int64)
    ids = np.concatenate([np.arange(N), np.sort(rng.choice(N, 9000, replace=False))]).astype(np.int32)
    g = vf.Index(X, off, ids, 1 << 30, 8)
    o = oracle.Index(X, off, ids, 1 << 30, 8)
    Q, qoff, qlab = _queries(dim, 150, [0, 1], seed=4)
    a, ad = g.search(Q, qoff, qlab, k=10, exact=True)
    e, ed = o.exact_knn(Q, qoff, qlab, k=10)
    assert (a == e).all() and (ad == ed.astype(np.float32)).all()
    st = g.last_stats()
    assert st["n_tiles"] > st["n_segments"]


@pytest.mark.parametrize("store", ["u8", "tf32"])
@pytest.mark.parametrize("dim", [4, 32, 48, 128])
def test_f32int_scan_exact(vf, dim, store):
    """Integer-valued fp32: values in [0, 255] are kept as a lossless u8 row store (kind::i8);
    other integers in the tf32-exact range run kind::tf32, whose products and partial sums are
    exact. Either way ids and distances are bit-identical to the fp32 oracle."""
    X8, off, ids = _u8_scan_index(dim, seed=dim + 1)
    shift = 0 if store == "u8" else 128
    X = X8.astype(np.float32) - shift
    g = vf.Index(X, off, ids, 1 << 30, 8)
    info = g.info()
    assert info["bytes_norms"] > 0                  # the tensor-core scan is enabled for this index
    assert (info["bytes_u8_store"] > 0) == (store == "u8")
    o = oracle.Index(X, off, ids, 1 << 30, 8)
    Q8, qoff, qlab = _queries(dim, 500, np.arange(len(off) - 1), seed=dim + 2)
    Q = Q8.astype(np.float32) - shift
    for k in (1, 10, 40):
        a, ad = g.search(Q, qoff, qlab, k=k, itopk=max(k, 16))
        e, ed = o.exact_knn(Q, qoff, qlab, k=k)
        assert (a == e).all() and (ad == ed.astype(np.float32)).all(), (dim, k)


@pytest.mark.parametrize("store", ["u8", "tf32"])
def test_f32_non_integral_query_falls_back(vf, store):
    """A batch holding a query outside the fast path's exact range runs the fp32 FFMA kernels
    instead: the integral queries stay bit-exact, the others within the generic-fp32 tolerance."""
    dim = 32
    X8, off, ids = _u8_scan_index(dim, seed=3)
    X = X8.astype(np.float32) - (0 if store == "u8" else 128)
    g = vf.Index(X, off, ids, 1 << 30, 8)
    o = oracle.Index(X, off, ids, 1 << 30, 8)
    Q8, qoff, qlab = _queries(dim, 200, np.arange(len(off) - 1), seed=8)
    Q = Q8.astype(np.float32)
    Q[17, 3] += 0.5
    Q[40, 0] = 5000.0                                # integral but above the tf32-exact bound
    a, ad = g.search(Q, qoff, qlab, k=10, itopk=16)
    e, ed = o.exact_knn(Q, qoff, qlab, k=10)
    ok = np.ones(len(Q), bool)
    ok[[17, 40]] = False
    assert (a[ok] == e[ok]).all() and (ad[ok] == ed[ok].astype(np.float32)).all()
    np.testing.assert_allclose(ad[~ok], ed[~ok], rtol=1e-5)
    # and the next all-integral batch is back on the tensor-core path, still exact
    b, bd = g.search(Q[ok], np.arange(ok.sum() + 1, dtype=np.int64), qlab[ok], k=10, itopk=16)
    assert (b == e[ok]).all() and (bd == ed[ok].astype(np.float32)).all()


def test_and_prefilter_pool_overflow_is_exact(vf, monkeypatch):
    """HS AND tiles are pre-filtered into a survivor pool; tiles that overflow it (or their piece
    list) are scanned in full. Either way the results equal Definition 1."""
    from workload import gen
    cfg, X, off, ids, go, gi = small_random_index(seed=21, N=6000, D=64, L=8, F=3.0, T=500, R=8,
                                                  dtype="u8")
    g = vf.Index(X, off, ids, cfg.threshold_T, cfg.degree_R, go, gi)
    o = oracle.Index(X, off, ids, cfg.threshold_T, cfg.degree_R, go, gi)
    Q = gen.gen_query_vectors(cfg, n=300)
    qoff, qlab = gen.gen_query_labels(cfg, off, ids, n=300, mode="and2")
    e, ed = o.exact_knn(Q, qoff, qlab, k=10, op="and")
    for cap in (None, "1", "300"):
        if cap is None:
            monkeypatch.delenv("VF_POOL_CAP", raising=False)
        else:
            monkeypatch.setenv("VF_POOL_CAP", cap)
        a, ad = g.search(Q, qoff, qlab, k=10, op="and", exact=True)
        assert (a == e).all() and (ad == ed.astype(np.float32)).all(), cap


@pytest.mark.parametrize("per_label", [1, 2, 3, 4, 5])
def test_u8_scan_few_queries_long_labels(vf, per_label):
    """1-5 queries per label over labels of 600-4000 rows (many 128-row stages): the regime where
    several epilogue warps share one query's rows (split selection, merged at the last stage)."""
    dim = 128
    X, off, ids = _u8_scan_index(dim, N=4000, seed=31)
    g = vf.Index(X, off, ids, 1 << 30, 8)
    o = oracle.Index(X, off, ids, 1 << 30, 8)
    labels = [5, 6, 7, 8]                            # 600, 1024, 1500, 4000 rows
    n = per_label * len(labels)
    Q, qoff, _ = _queries(dim, n, [0], seed=per_label)
    qlab = np.repeat(np.array(labels, np.int32), per_label)
    for k in (1, 10, 32):
        a, ad = g.search(Q, qoff, qlab, k=k, itopk=max(k, 16))
        e, ed = o.exact_knn(Q, qoff, qlab, k=k)
        assert (a == e).all() and (ad == ed.astype(np.float32)).all(), (per_label, k)


def test_u8_scan_mixed_query_group_sizes_exact_mode(vf):
    """Consecutive tiles alternating between split (<= 4 queries) and unsplit query groups, long
    labels, exact mode: the split lists are merged before any warp starts the next tile."""
    dim = 64
    rng = np.random.default_rng(17)
    N = 30000
    X = rng.integers(0, 256, size=(N, dim), dtype=np.uint8)
    sizes = [9000, 5000, 12000, 700, 3000, 20000, 150]
    ids = [np.sort(rng.choice(N, size=s_, replace=False)).astype(np.int32) for s_ in sizes]
    off = np.zeros(len(sizes) + 1, np.int64)
    off[1:] = np.cumsum(sizes)
    ids = np.concatenate(ids)
    g = vf.Index(X, off, ids, 1 << 30, 8)
    o = oracle.Index(X, off, ids, 1 << 30, 8)
    per = [1, 40, 2, 3, 70, 4, 9]                    # queries per label
    qlab = np.repeat(np.arange(len(sizes), dtype=np.int32), per)
    Q, qoff, _ = _queries(dim, len(qlab), [0], seed=23)
    e, ed = o.exact_knn(Q, qoff, qlab, k=10)
    for ex in (False, True):
        a, ad = g.search(Q, qoff, qlab, k=10, itopk=16, exact=ex)
        assert (a == e).all() and (ad == ed.astype(np.float32)).all(), ex


@pytest.mark.parametrize("op", ["single", "and"])
def test_small_query_groups_are_exact(vf, op):
    """Tiles of few queries on short lists (the YFCC-shaped mix): single and AND, normal and
    exact mode, bit-exact against the oracle."""
    from workload import gen
    cfg, X, off, ids, go, gi = small_random_index(seed=41, N=5000, D=96, L=12, F=2.5, T=800, R=8,
                                                  dtype="u8")
    g = vf.Index(X, off, ids, cfg.threshold_T, cfg.degree_R, go, gi)
    o = oracle.Index(X, off, ids, cfg.threshold_T, cfg.degree_R, go, gi)
    Q = gen.gen_query_vectors(cfg, n=300)
    if op == "single":
        qoff = np.arange(301, dtype=np.int64)
        qlab = np.random.default_rng(2).integers(0, cfg.n_labels, size=300).astype(np.int32)
    else:
        qoff, qlab = gen.gen_query_labels(cfg, off, ids, n=300, mode="and2")
    for exact in (False, True):
        a, ad = g.search(Q, qoff, qlab, k=10, itopk=32, op=op, exact=exact)
        e, ed = (o.exact_knn(Q, qoff, qlab, k=10, op=op) if exact else
                 o.search(Q, qoff, qlab, k=10, itopk=32, op=op))
        assert (a == e).all() and (ad == ed.astype(np.float32)).all(), exact


@pytest.mark.parametrize("cap", [None, "1", "700"])
@pytest.mark.parametrize("exact", [False, True])
def test_and_prefilter_mixed_and_compacted_tiles(vf, monkeypatch, cap, exact):
    """k_and_filter (P:L559 'before distance'): tiles whose queries all carry an AND predicate are
    compacted to the rows passing some query (pass bits per survivor); tiles mixing single-label
    and AND queries keep every row with per-row pass bits; a full pool leaves the tile to the
    scan's own verification. All three bit-exact vs the oracle, greedy and parallel policies."""
    from workload import gen
    if cap is None:
        monkeypatch.delenv("VF_POOL_CAP", raising=False)
    else:
        monkeypatch.setenv("VF_POOL_CAP", cap)
    cfg, X, off, ids, go, gi = small_random_index(seed=27, N=8000, D=64, L=10, F=3.0, T=700, R=8,
                                                  dtype="u8")
    g = vf.Index(X, off, ids, cfg.threshold_T, cfg.degree_R, go, gi)
    o = oracle.Index(X, off, ids, cfg.threshold_T, cfg.degree_R, go, gi)
    Q = gen.gen_query_vectors(cfg, n=400)
    qoff, qlab = gen.gen_query_labels(cfg, off, ids, n=400, mode="mix_and")
    for mode in ("greedy", "parallel"):
        a, ad = g.search(Q, qoff, qlab, k=10, itopk=32, op="and", recall_mode=mode, exact=exact)
        if exact:
            e, ed = o.exact_knn(Q, qoff, qlab, k=10, op="and")
        else:
            e, ed = o.search(Q, qoff, qlab, k=10, itopk=32, op="and", recall_mode=mode)
        assert (a == e).all() and (ad == ed.astype(np.float32)).all(), (mode, cap, exact)


def test_and_prefilter_wide_label_union(vf):
    """AND3 queries sharing their smallest label: one segment's other labels exceed the 64 bit
    positions of the pre-filter's label union, which then verifies per query; results equal
    Definition 1 (every label LS, so greedy AND is exact)."""
    rng = np.random.default_rng(77)
    N, dim = 6000, 64
    X = rng.integers(0, 256, size=(N, dim), dtype=np.uint8)
    lists = [np.sort(rng.choice(N, size=400, replace=False))]
    lists += [np.sort(rng.choice(N, size=2500, replace=False)) for _ in range(120)]
    off = np.zeros(len(lists) + 1, np.int64)
    off[1:] = np.cumsum([len(x) for x in lists])
    ids = np.concatenate(lists).astype(np.int32)
    T = 1 << 30
    g = vf.Index(X, off, ids, T, 8)
    o = oracle.Index(X, off, ids, T, 8)
    n = 130                                          # > 64: the batched path (k_and_filter)
    Q = rng.integers(0, 256, size=(n, dim), dtype=np.uint8)
    labs = [np.array([0] + list(rng.choice(np.arange(1, 121), size=2, replace=False)), np.int32) for _ in range(n)]
    qoff = np.zeros(n + 1, np.int64)
    qoff[1:] = np.cumsum([len(x) for x in labs])
    qlab = np.concatenate(labs)
    for k in (1, 10):
        a, ad = g.search(Q, qoff, qlab, k=k, itopk=16, op="and")
        e, ed = o.exact_knn(Q, qoff, qlab, k=k, op="and")
        assert (a == e).all() and (ad == ed.astype(np.float32)).all(), k


@pytest.mark.parametrize("mode", ["single", "mix_and", "and2"])
def test_tile_packing_is_exact(vf, monkeypatch, mode):
    """k_pack: small single-tile segments share one tensor-core tile (rows carry their own
    segment's pass bits). Results bit-identical with packing off and on, and to the oracle."""
    from workload import gen
    cfg, X, off, ids, go, gi = small_random_index(seed=51, N=20000, D=192, L=60, F=4.0, T=1500, R=8, dtype="u8")
    g = vf.Index(X, off, ids, cfg.threshold_T, cfg.degree_R, go, gi)
    o = oracle.Index(X, off, ids, cfg.threshold_T, cfg.degree_R, go, gi)
    Q = gen.gen_query_vectors(cfg, n=600)
    qoff, qlab = gen.gen_query_labels(cfg, off, ids, n=600, mode=mode)
    op = "single" if mode == "single" else "and"
    res = {}
    for pack in ("0", "1"):
        monkeypatch.setenv("VF_PACK", pack)
        res[pack] = g.search(Q, qoff, qlab, k=10, itopk=32, op=op)
        assert g.last_stats()["n_scan_items"] > 100
    assert (res["0"][0] == res["1"][0]).all() and (res["0"][1] == res["1"][1]).all()
    e, ed = o.search(Q, qoff, qlab, k=10, itopk=32, op=op)
    assert (res["1"][0] == e).all() and (res["1"][1] == ed.astype(np.float32)).all()



@pytest.mark.parametrize("cap", [None, "6000"])
def test_f3_tile_sizes_are_exact(vf, monkeypatch, cap):
    """Segments scanned only through f3 AND routing (every tile compacted by the AND pre-filter)
    use large tiles (VF_F3_TILE rows): a tile's survivors come in up to kMaxPieces pieces, more
    survivors than that leave the tile to the scan's own verification, and a small survivor pool
    leaves tiles uncompacted. Results bit-identical across tile sizes, and to the oracle (greedy
    AND with f3 routing; Definition 1 in exact mode, where tiles keep the normal size)."""
    from workload import gen
    if cap is None:
        monkeypatch.delenv("VF_POOL_CAP", raising=False)
    else:
        monkeypatch.setenv("VF_POOL_CAP", cap)
    cfg, X, off, ids, go, gi = small_random_index(seed=61, N=40000, D=64, L=12, F=3.0, T=1500, R=8,
                                                  dtype="u8")
    assert np.diff(off).max() > 4 * 4096           # multi-tile segments at every tile size
    g = vf.Index(X, off, ids, cfg.threshold_T, cfg.degree_R, go, gi)
    o = oracle.Index(X, off, ids, cfg.threshold_T, cfg.degree_R, go, gi)
    Q = gen.gen_query_vectors(cfg, n=500)
    qoff, qlab = gen.gen_query_labels(cfg, off, ids, n=500, mode="mix_and")
    thr = 10 ** 7                                      # every greedy AND item with an HS l* is scanned
    for exact in (False, True):
        res = {}
        for rows in ("2048", "8192", "32768"):
            monkeypatch.setenv("VF_F3_TILE", rows)
            res[rows] = g.search(Q, qoff, qlab, k=10, itopk=32, op="and", exact=exact, and_scan_threshold=thr)
        for rows in ("8192", "32768"):
            assert (res[rows][0] == res["2048"][0]).all() and (res[rows][1] == res["2048"][1]).all(), (exact, rows)
        if exact:
            e, ed = o.exact_knn(Q, qoff, qlab, k=10, op="and")
        else:
            e, ed = o.search(Q, qoff, qlab, k=10, itopk=32, op="and", and_scan_threshold=thr)
        assert (res["8192"][0] == e).all() and (res["8192"][1] == ed.astype(np.float32)).all(), (exact, cap)
