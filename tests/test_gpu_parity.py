"""GPU path (through the C-ABI) vs the CPU oracle, element by element on the same seeded inputs.

Bar (BASELINE.json north_star): integer-valued data (u8, fp32-int) -> ids and
distances bit-exact on both paths, and per-item V/E counters identical on the graph path;
generic fp32 -> scan distances within 1e-5 relative, ids identical outside tie bands, graph
results overlap >= 0.99.
"""
import numpy as np
import pytest

import oracle
from conftest import golden, small_random_index

pytestmark = pytest.mark.gpu


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


def _pair(vf, X, w, go, gi, T=None, R=None):
    T = T or w.cfg.threshold_T
    R = R or w.cfg.degree_R
    g = vf.Index(X, w.post_off, w.post_ids, T, R, go, gi)
    o = oracle.Index(X, w.post_off, w.post_ids, T, R, go, gi)
    return g, o


def _items_match(g, o_ctr):
    """GPU per-item (label, path, V, E) equal the oracle's (canonical item order)."""
    rec = g.last_items()
    exp = []
    for i in range(o_ctr.shape[0]):
        for t in range(o_ctr.shape[1]):
            if o_ctr[i, t, 0] >= 0:
                exp.append((i, o_ctr[i, t, 0], o_ctr[i, t, 1], o_ctr[i, t, 2], o_ctr[i, t, 3]))
    got = [(r[0], r[1], r[2], r[3], r[4]) for r in rec]
    assert len(got) == len(exp)
    bad = [(a, b) for a, b in zip(got, exp) if a != b]
    assert not bad, bad[:5]


@pytest.mark.parametrize("dtype", ["f32int", "u8"])
@pytest.mark.parametrize("itopk", [16, 20, 28, 32, 40, 56, 64, 100, 128, 160])
def test_single_label_bit_exact(vf, tiny, dtype, itopk):
    w, go, gi = tiny
    X, Q = _variant(tiny, dtype)
    g, o = _pair(vf, X, w, go, gi)
    ids, d = g.search(Q, w.q_off, w.q_lab, k=10, itopk=itopk)
    oi, od, octr = o.search(Q, w.q_off, w.q_lab, k=10, itopk=itopk, counters=True)
    assert (ids == oi).all()
    assert (d == od.astype(np.float32)).all()
    _items_match(g, octr)
    st = g.last_stats()
    assert st["n_graph_items"] > 400 and st["n_scan_items"] > 300


def test_single_label_generic_float(vf, tiny):
    w, go, gi = tiny
    X, Q = _variant(tiny, "f32float")
    g, o = _pair(vf, X, w, go, gi)
    ids, d = g.search(Q, w.q_off, w.q_lab, k=10, itopk=64)
    oi, od, octr = o.search(Q, w.q_off, w.q_lab, k=10, itopk=64, counters=True)
    scan = octr[:, 0, 1] == oracle.PATH_SCAN
    fin = np.isfinite(od)
    np.testing.assert_allclose(d[fin], od[fin], rtol=1e-5, atol=1e-7)
    # scan rows: identical ids except swaps inside a 1e-5 tie band
    for i in np.flatnonzero(scan):
        diff = ids[i] != oi[i]
        if diff.any():
            band = np.abs(od[i][diff] - od[i][np.argmax(diff)]) <= 1e-5 * od[i][diff]
            assert band.all()
    overlap = np.mean([np.intersect1d(ids[i], oi[i]).size / 10 for i in np.flatnonzero(~scan)])
    assert overlap >= 0.99


@pytest.mark.parametrize("op,mode", [("and", "greedy"), ("and", "parallel"), ("or", "greedy")])
@pytest.mark.parametrize("dtype", ["f32int", "u8"])
def test_multilabel_bit_exact(vf, tiny, op, mode, dtype):
    from workload import gen
    w, go, gi = tiny
    X, Q = _variant(tiny, dtype)
    qoff, qlab = gen.gen_query_labels(w.cfg, w.post_off, w.post_ids, n=len(Q),
                                      mode="and2" if op == "and" else "or2")
    g, o = _pair(vf, X, w, go, gi)
    ids, d = g.search(Q, qoff, qlab, k=10, itopk=32, op=op, recall_mode=mode)
    oi, od, octr = o.search(Q, qoff, qlab, k=10, itopk=32, op=op, recall_mode=mode, counters=True)
    assert (ids == oi).all()
    assert (d == od.astype(np.float32)).all()
    _items_match(g, octr)


@pytest.mark.parametrize("op", ["single", "and", "or"])
def test_exact_mode_is_definition1(vf, tiny, op):
    """exact=1 (T = inf) equals the oracle's brute-force Definition-1 ground truth."""
    from workload import gen
    w, go, gi = tiny
    qoff, qlab = (w.q_off, w.q_lab) if op == "single" else \
        gen.gen_query_labels(w.cfg, w.post_off, w.post_ids, n=len(w.Q), mode=op + "2")
    g, o = _pair(vf, w.X, w, go, gi)
    ids, d = g.search(w.Q, qoff, qlab, k=10, op=op, exact=True)
    gt, gd = o.exact_knn(w.Q, qoff, qlab, k=10, op=op)
    assert (ids == gt).all()
    assert (d == gd.astype(np.float32)).all()


def test_exact_mode_multi_tile(vf):
    """Labels longer than one scan tile (4096 rows): partial lists merged exactly."""
    from workload import gen, graphs
    cfg = gen.config("tiny", n_points=30000, n_labels=6, threshold_T=100000)
    X = gen.gen_vectors(cfg)
    off, ids_ = gen.gen_postings(cfg)
    assert np.diff(off).max() > 8192
    Q = gen.gen_query_vectors(cfg, n=300)
    qoff, qlab = gen.gen_query_labels(cfg, off, ids_, n=300, mode="single")
    g = vf.Index(X, off, ids_, cfg.threshold_T, 16)
    o = oracle.Index(X, off, ids_, cfg.threshold_T, 16)
    r_ids, r_d = g.search(Q, qoff, qlab, k=10)
    e_ids, e_d = o.exact_knn(Q, qoff, qlab, k=10)
    assert (r_ids == e_ids).all() and (r_d == e_d.astype(np.float32)).all()
    assert g.last_stats()["n_tiles"] > g.last_stats()["n_segments"]


def test_edge_cases(vf):
    """Empty / unknown labels, zero-label queries, k > |C_l|, k = itopk, S = 1, ragged sizes."""
    cfg, X, off, ids_, go, gi = small_random_index(seed=31, N=500, L=14, T=30, R=8)
    sizes = np.diff(off)
    # make label 0 a single-point HS label by hand is impossible at T=30; use T=1 index below
    g = vf.Index(X, off, ids_, cfg.threshold_T, cfg.degree_R, go, gi)
    o = oracle.Index(X, off, ids_, cfg.threshold_T, cfg.degree_R, go, gi)
    rng = np.random.default_rng(0)
    n = 64
    Q = rng.integers(0, 256, size=(n, cfg.dim)).astype(np.float32)
    counts = rng.integers(0, 4, size=n)
    qoff = np.zeros(n + 1, np.int64)
    qoff[1:] = np.cumsum(counts)
    qlab = rng.integers(-2, cfg.n_labels + 3, size=int(qoff[-1])).astype(np.int32)
    for op, mode in [("or", "greedy"), ("and", "greedy"), ("and", "parallel")]:
        for k, itopk in [(1, 1), (7, 7), (40, 64)]:
            a, ad = g.search(Q, qoff, qlab, k=k, itopk=itopk, op=op, recall_mode=mode)
            b, bd = o.search(Q, qoff, qlab, k=k, itopk=itopk, op=op, recall_mode=mode)
            assert (a == b).all(), (op, mode, k)
            assert (ad == bd.astype(np.float32)).all()
    assert sizes.min() >= 0


def test_single_point_and_tiny_labels(vf):
    """T = 1: every label is HS, including |C_l| = 1 and |C_l| <= R."""
    X = np.array([[0, 0], [3, 4], [6, 8], [1, 1], [9, 9]], np.float32)
    off = np.array([0, 1, 3, 5], np.int64)
    ids_ = np.array([2, 0, 1, 3, 4], np.int32)
    goff = np.array([0, 1, 3, 5], np.int64)
    R = 4
    gids = np.full(5 * R, -1, np.int32)
    gids[1 * R] = 1; gids[2 * R] = 0; gids[3 * R] = 1; gids[4 * R] = 0
    g = vf.Index(X, off, ids_, 1, R, goff, gids)
    o = oracle.Index(X, off, ids_, 1, R, goff, gids)
    Q = np.array([[0, 0], [5, 5], [2, 2]], np.float32)
    qoff = np.arange(4, dtype=np.int64)
    for lab in range(3):
        ql = np.full(3, lab, np.int32)
        a, ad = g.search(Q, qoff, ql, k=3, itopk=4)
        b, bd = o.search(Q, qoff, ql, k=3, itopk=4)
        assert (a == b).all() and (ad == bd.astype(np.float32)).all()


def test_appendix_b_trace_on_gpu(vf):
    """The hand-derived beam trace (tests/golden/beam_appendix_b.json) on the GPU kernel: the
    seed is chosen so the content-keyed sampler's single entry is local id 0."""
    gb = golden("beam_appendix_b.json")
    pts = np.array(gb["points_1d"], np.float32)
    X = np.zeros((len(pts), 4), np.float32)
    X[:, 0] = pts
    rows = np.array(gb["rows"], np.int32)
    off = np.array([0, len(pts)], np.int64)
    ids_ = np.arange(len(pts), dtype=np.int32)
    goff = np.array([0, len(pts)], np.int64)
    g = vf.Index(X, off, ids_, len(pts), 2, goff, rows.reshape(-1))
    q = np.zeros((1, 4), np.float32)
    q[0, 0] = gb["query_1d"]
    qh = oracle.query_hash(q[0])
    seed = next(s for s in range(1000) if oracle.entry_hash(s, qh, 0, 0, len(pts)) == 0)
    a, ad = g.search(q, np.array([0, 1], np.int64), np.array([0], np.int32), k=2, itopk=2, n_init=1,
                     max_iterations=100, seed=seed)
    e = gb["expected"]
    assert a[0].tolist() == e["ids"] and ad[0].tolist() == e["dists"]
    rec = g.last_items()
    assert rec[0, 3] == e["V"] and rec[0, 4] == e["E"]


def test_device_buffers_and_stream_match_host(vf, tiny):
    import torch
    w, go, gi = tiny
    g = vf.Index(w.X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi)
    hi, hd = g.search(w.Q, w.q_off, w.q_lab, k=10, itopk=48)
    s = torch.cuda.Stream()
    Q, qo, ql = (torch.from_numpy(a).cuda() for a in (w.Q, w.q_off, w.q_lab))
    ids = torch.empty((len(w.Q), 10), dtype=torch.int32, device="cuda")
    d = torch.empty((len(w.Q), 10), dtype=torch.float32, device="cuda")
    g.search_into(Q, qo, ql, ids, d, k=10, itopk=48, stream=s)
    s.synchronize()
    assert (ids.cpu().numpy() == hi).all() and (d.cpu().numpy() == hd).all()


def test_batch_order_independence(vf, tiny):
    w, go, gi = tiny
    g = vf.Index(w.X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi)
    a, ad = g.search(w.Q, w.q_off, w.q_lab, k=10, itopk=32)
    perm = np.random.default_rng(1).permutation(len(w.Q))[:257]
    b, bd = g.search(w.Q[perm], np.arange(258, dtype=np.int64), w.q_lab[perm], k=10, itopk=32)
    assert (a[perm] == b).all() and (ad[perm] == bd).all()


@pytest.mark.parametrize("knobs", ["11", "139"])
def test_visited_overflow_to_global_table(vf, tiny, knobs, monkeypatch):
    """itopk large enough that the shared-memory visited set spills (139: hash table only -- the
    tiny labels otherwise take the visited bitmap, which never spills): still bit-exact."""
    monkeypatch.setenv("VF_KNOBS", knobs)
    w, go, gi = tiny
    g, o = _pair(vf, w.X, w, go, gi)
    ids, d = g.search(w.Q[:200], w.q_off[:201], w.q_lab[:w.q_off[200]], k=10, itopk=1024)
    oi, od = o.search(w.Q[:200], w.q_off[:201], w.q_lab[:w.q_off[200]], k=10, itopk=1024)
    assert (ids == oi).all() and (d == od.astype(np.float32)).all()
    assert g.last_stats()["graph_V_max"] > 512


def test_byte_accounting(vf, tiny):
    """Built-index bytes = the layout formula; RB keeps one copy of X."""
    w, go, gi = tiny
    g = vf.Index(w.X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi)
    info = g.info()
    sizes = np.diff(w.post_off)
    hs = sizes[sizes >= w.cfg.threshold_T].sum()
    ls = sizes[(sizes > 0) & (sizes < w.cfg.threshold_T)].sum()
    rb = info["row_bytes"]
    assert info["hs_rows"] == hs and info["ls_rows"] == ls
    assert info["bytes_vectors"] == w.cfg.n_points * rb
    assert info["bytes_graph"] == hs * w.cfg.degree_R * 8      # (local, global) edge pairs
    ls_sizes = sizes[(sizes > 0) & (sizes < w.cfg.threshold_T)]
    ls_pad = int(((ls_sizes + 3) // 4 * 4).sum())                 # 4-row aligned label bases
    assert info["bytes_ls_vectors"] == ls_pad * rb
    # redundancy bypassing saves exactly the HS vector copies
    assert info["bytes_total"] < info["bytes_total"] + hs * rb


@pytest.mark.parametrize("shards", [2, 3, 4])
@pytest.mark.parametrize("op,mode", [("single", "greedy"), ("and", "greedy"), ("and", "parallel"), ("or", "greedy")])
def test_virtual_shards_bit_identical(vf, tiny, shards, op, mode):
    """Label sharding (§8(e)) on one device: route -> ship items to owners -> execute -> return ->
    merge gives exactly the unsharded results (items are independent, the sampler keys on content)."""
    from workload import gen
    w, go, gi = tiny
    qoff, qlab = (w.q_off, w.q_lab) if op == "single" else \
        gen.gen_query_labels(w.cfg, w.post_off, w.post_ids, n=len(w.Q), mode="and2" if op == "and" else "or2")
    one = vf.Index(w.X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi)
    many = vf.Index(w.X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi, virtual_shards=shards)
    for itopk in (16, 64):
        a, ad = one.search(w.Q, qoff, qlab, k=10, itopk=itopk, op=op, recall_mode=mode)
        b, bd = many.search(w.Q, qoff, qlab, k=10, itopk=itopk, op=op, recall_mode=mode)
        assert (a == b).all() and (ad == bd).all()
    a, ad = one.search(w.Q, qoff, qlab, k=10, op=op, recall_mode=mode, exact=True)
    b, bd = many.search(w.Q, qoff, qlab, k=10, op=op, recall_mode=mode, exact=True)
    assert (a == b).all() and (ad == bd).all()
    info = many.info()
    assert info["owned_labels"] == one.info()["owned_labels"]      # every label owned exactly once


@pytest.mark.parametrize("thr", [0, 60, 400, 2**30])
def test_and_scan_routing_f3_bit_exact(vf, tiny, thr):
    """Selectivity-aware AND routing (f3): same fp64 decision on both sides, results bit-exact."""
    from workload import gen
    w, go, gi = tiny
    qoff, qlab = gen.gen_query_labels(w.cfg, w.post_off, w.post_ids, n=len(w.Q), mode="and2")
    g, o = _pair(vf, w.X, w, go, gi)
    ids, d = g.search(w.Q, qoff, qlab, k=10, itopk=32, op="and", and_scan_threshold=thr)
    oi, od, octr = o.search(w.Q, qoff, qlab, k=10, itopk=32, op="and", and_scan_threshold=thr, counters=True)
    assert (ids == oi).all() and (d == od.astype(np.float32)).all()
    _items_match(g, octr)


def test_u8_store_fallback_batch(vf, tiny):
    """Integer-valued fp32 is served from the lossless u8 row store; a batch holding a fractional
    query runs the fp32 kernels on both paths: every other query stays bit-exact."""
    w, go, gi = tiny
    g, o = _pair(vf, w.X, w, go, gi)
    assert g.info()["bytes_u8_store"] > 0
    Q = w.Q.copy()
    Q[5, 0] += 0.25
    ids, d = g.search(Q, w.q_off, w.q_lab, k=10, itopk=32)
    oi, od = o.search(Q, w.q_off, w.q_lab, k=10, itopk=32)
    keep = np.arange(len(Q)) != 5
    assert (ids[keep] == oi[keep]).all() and (d[keep] == od[keep].astype(np.float32)).all()
    assert g.last_stats()["row_bytes"] == (w.X.shape[1] * 4 + 15) // 16 * 16     # the fp32 rows ran
    assert np.intersect1d(ids[5], oi[5]).size >= 9


@pytest.mark.parametrize("thr", [0, 500, 1500, 3000, 2**31 - 1])
def test_scan_threshold_f2_bit_exact(vf, tiny, thr):
    """Search-time specificity threshold (f2): labels below max(T, T') are scanned on both sides;
    results and per-item counters identical for single and greedy-AND queries."""
    from workload import gen
    w, go, gi = tiny
    g, o = _pair(vf, w.X, w, go, gi)
    ids, d = g.search(w.Q, w.q_off, w.q_lab, k=10, itopk=32, scan_threshold=thr)
    oi, od, octr = o.search(w.Q, w.q_off, w.q_lab, k=10, itopk=32, scan_threshold=thr, counters=True)
    assert (ids == oi).all() and (d == od.astype(np.float32)).all()
    _items_match(g, octr)
    qoff, qlab = gen.gen_query_labels(w.cfg, w.post_off, w.post_ids, n=len(w.Q), mode="and2")
    ids, d = g.search(w.Q, qoff, qlab, k=10, itopk=32, op="and", scan_threshold=thr)
    oi, od = o.search(w.Q, qoff, qlab, k=10, itopk=32, op="and", scan_threshold=thr)
    assert (ids == oi).all() and (d == od.astype(np.float32)).all()


@pytest.mark.parametrize("density", ["0", "4", "256", "1024"])
def test_label_bitmaps_do_not_change_results(vf, tiny, density, monkeypatch):
    """Membership bitmaps of the largest labels (predicate fast path, read at build time): none
    (0), only labels with >= N/4 points (4: a mix of bitmap and label-list checks inside one query),
    all labels with >= N/256 or N/1024 points (1024, the default). AND / OR results and per-item counters
    stay bit-identical to the oracle, which has no bitmaps."""
    from workload import gen
    monkeypatch.setenv("VF_BITMAP_DENSITY", density)
    w, go, gi = tiny
    g, o = _pair(vf, w.X, w, go, gi)
    for mode_q, op, mode in [("and2", "and", "greedy"), ("and2", "and", "parallel"), ("or2", "or", "greedy")]:
        qoff, qlab = gen.gen_query_labels(w.cfg, w.post_off, w.post_ids, n=len(w.Q), mode=mode_q)
        for thr in (0, 400):
            ids, d = g.search(w.Q, qoff, qlab, k=10, itopk=32, op=op, recall_mode=mode, and_scan_threshold=thr)
            oi, od, octr = o.search(w.Q, qoff, qlab, k=10, itopk=32, op=op, recall_mode=mode,
                                    and_scan_threshold=thr, counters=True)
            assert (ids == oi).all() and (d == od.astype(np.float32)).all(), (op, mode, thr)
            _items_match(g, octr)


def test_kernel_activity_spans(vf, tiny):
    """vf_get_last_stats reports the scan / graph kernels' device-clock spans; they are positive
    when the kernel ran and fit inside the whole search."""
    w, go, gi = tiny
    g = vf.Index(w.X, w.post_off, w.post_ids, w.cfg.threshold_T, w.cfg.degree_R, go, gi)
    g.set_profiling(True)
    g.search(w.Q, w.q_off, w.q_lab, k=10, itopk=32)
    st = g.last_stats()
    assert st["n_graph_items"] > 0 and st["ms_graph_active"] > 0
    assert st["ms_graph_active"] <= st["ms_total"] + 1e-3
    if st["n_scan_items"] > 0 and g.info()["bytes_norms"] > 0:     # tensor-core scan ran
        assert 0 < st["ms_scan_active"] <= st["ms_total"] + 1e-3


@pytest.mark.parametrize("w_", [3, 4])
@pytest.mark.parametrize("op,mode", [("single", "greedy"), ("and", "greedy"), ("and", "parallel")])
@pytest.mark.parametrize("itopk", [64, 384])
def test_search_width_3_4_bit_exact(vf, tiny, w_, op, mode, itopk):
    """w * R > 32: more than one 32-child batch per iteration and n_init = w * R entries in two
    batches (reading #37); the oracle's multi-parent rule is pinned by
    tests/golden/beam_multi_parent.json. ids, distances and per-item V / E identical."""
    from workload import gen
    w, go, gi = tiny
    X, Q = _variant(tiny, "u8")
    if op == "single":
        qoff, qlab = w.q_off, w.q_lab
    else:
        qoff, qlab = gen.gen_query_labels(w.cfg, w.post_off, w.post_ids, n=len(Q), mode="and2")
    g, o = _pair(vf, X, w, go, gi)
    ids, d = g.search(Q, qoff, qlab, k=10, itopk=itopk, search_width=w_, op=op, recall_mode=mode)
    oi, od, octr = o.search(Q, qoff, qlab, k=10, itopk=itopk, search_width=w_, op=op, recall_mode=mode,
                            counters=True)
    assert (ids == oi).all()
    assert (d == od.astype(np.float32)).all()
    _items_match(g, octr)


def test_device_offsets_invalid_queries_get_empty_rows(vf, tiny):
    """Device offset arrays are checked on the device (include/vf.h n_query_labels): a query with
    more than 64 labels, or whose offsets leave [0, n_query_labels), gets an empty row and is
    counted in n_invalid_queries; the other queries are answered as usual. Both the per-query
    path (<= 64 queries) and the batched path."""
    import torch
    w, go, gi = tiny
    g, o = _pair(vf, w.X, w, go, gi)
    for n in (40, 120):
        Q = w.Q[:n]
        qoff = w.q_off[:n + 1].copy()
        qlab = w.q_lab[:qoff[-1]].copy()
        oi, od = o.search(Q, qoff, qlab, k=10, itopk=32)
        # query 5 carries its label 70 times (> 64 labels)
        extra = 69
        qlab = np.concatenate([qlab[:qoff[6]], np.full(extra, qlab[qoff[5]], np.int32), qlab[qoff[6]:]])
        qoff[6:] += extra
        # query 9 ends beyond the label array (and so query 10 starts after it ends)
        qoff[10] = 10 ** 9
        bad = {5, 9, 10}
        ids = torch.empty((n, 10), dtype=torch.int32, device="cuda")
        dd = torch.empty((n, 10), dtype=torch.float32, device="cuda")
        g.search_into(torch.from_numpy(Q).cuda(), torch.from_numpy(qoff).cuda(), torch.from_numpy(qlab).cuda(),
                      ids, dd, k=10, itopk=32, n_query_labels=int(qlab.size))
        torch.cuda.synchronize()
        st = g.last_stats()
        ids, dd = ids.cpu().numpy(), dd.cpu().numpy()
        assert st["n_invalid_queries"] == len(bad), (n, st["n_invalid_queries"])
        for i in range(n):
            if i in bad:
                assert (ids[i] == -1).all() and np.isinf(dd[i]).all(), (n, i)
            else:
                assert (ids[i] == oi[i]).all() and (dd[i] == od[i].astype(np.float32)).all(), (n, i)


@pytest.mark.parametrize("knobs", ["0", "11", "16", "43", "75", "139", "203"])
def test_implementation_switches_do_not_change_results(vf, tiny, knobs, monkeypatch):
    """VF_KNOBS (reading #52; read per search) selects equal-result implementation
    variants: signature loads in the AND pre-filter, graph row / adjacency prefetch, pre-filter
    occupancy, next-parent adjacency prefetch, the visited set's one-probe / two-phase / bitmap
    paths. Every setting returns the oracle's ids, distances and per-item V / E (itopk 512 makes
    the hash-table settings spill to the global table)."""
    from workload import gen
    monkeypatch.setenv("VF_KNOBS", knobs)
    w, go, gi = tiny
    g, o = _pair(vf, w.X, w, go, gi)
    for mode_q, op, mode, thr in [("single", "single", "greedy", 0), ("and2", "and", "greedy", 400),
                                   ("and2", "and", "parallel", 0), ("or2", "or", "greedy", 0)]:
        if mode_q == "single":
            qoff, qlab = w.q_off, w.q_lab
        else:
            qoff, qlab = gen.gen_query_labels(w.cfg, w.post_off, w.post_ids, n=len(w.Q), mode=mode_q)
        for itopk in (32, 512):
            ids, d = g.search(w.Q, qoff, qlab, k=10, itopk=itopk, op=op, recall_mode=mode, and_scan_threshold=thr,
                              search_width=2)
            oi, od, octr = o.search(w.Q, qoff, qlab, k=10, itopk=itopk, op=op, recall_mode=mode,
                                    and_scan_threshold=thr, search_width=2, counters=True)
            assert (ids == oi).all() and (d == od.astype(np.float32)).all(), (knobs, op, mode, itopk)
            _items_match(g, octr)
