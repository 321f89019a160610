"""CPU oracle for the label-filtered top-k search path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package. It wraps oracle/oracle.c (plain C, scalar loops, fp64/int64 arithmetic) via
ctypes and adds recall@K in plain numpy. It shares no code with the CUDA
library in paper_2506_00812_b200/.

Parity status per function: every function below is pinned by tests in
tests/test_oracle_*.py; "absolute recall level" of the beam search on a given graph is
"parity unpinned" (it depends on the input graph).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

OP = {"single": 0, "or": 1, "and": 2}
RECALL_MODE = {"greedy": 0, "parallel": 1}
PATH_NONE, PATH_SCAN, PATH_GRAPH = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc, no fast-math, no FP contraction: reading #33)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-fno-fast-math", "-ffp-contract=off", "-fPIC", "-shared",
               "-pthread", "-o", _SO + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_SO + ".tmp", _SO)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        p, i32, i64, u32, d = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_double
        L.or_index_create.restype = p
        L.or_index_create.argtypes = [C.c_int, C.c_int, i64, p, i32, p, p, i32, i32, p, p]
        L.or_index_free.argtypes = [p]
        L.or_verify.restype = C.c_int
        L.or_verify.argtypes = [p, i64, i64, p, C.c_int, p]
        L.or_query_hash.restype = u32
        L.or_query_hash.argtypes = [C.c_int, C.c_int, p]
        L.or_entry_hash.restype = u32
        L.or_entry_hash.argtypes = [u32, u32, i32, u32, u32]
        L.or_route.restype = i64
        L.or_route.argtypes = [p, i64, p, p, C.c_int, C.c_int, C.c_int, i32, i32, p, i64, p]
        L.or_merge.argtypes = [C.c_int, C.c_int, p, p, p, p]
        L.or_search.restype = C.c_int
        L.or_search.argtypes = [p, i64, p, p, p, C.c_int, C.c_int, C.c_int, i32, i32, i32, i32,
                                i32, u32, i32, p, p, p, i32, C.c_int, i32, i32]
        L.or_exact_knn.restype = C.c_int
        L.or_exact_knn.argtypes = [p, i64, p, p, p, C.c_int, i32, p, p, C.c_int]
        L.or_label_knn.restype = C.c_int
        L.or_label_knn.argtypes = [p, i32, C.c_int, p]
        L.or_cagra_rows.restype = C.c_int
        L.or_cagra_rows.argtypes = [i64, C.c_int, p, C.c_int, p, p]
        L.or_index_pt_off.restype = i64
        L.or_index_pt_off.argtypes = [p, i64]
        L.or_index_pt_lab.restype = p
        L.or_index_pt_lab.argtypes = [p]
        for f in ("or_mem_hs_bytes", "or_mem_ls_bytes", "or_mem_single_bytes", "or_mem_map_bytes"):
            getattr(L, f).restype = d
        L.or_mem_hs_bytes.argtypes = [d, d, d, d, d]
        L.or_mem_ls_bytes.argtypes = [d, d, d, d]
        L.or_mem_single_bytes.argtypes = [d, d, d, d]
        L.or_mem_map_bytes.argtypes = [d, d, d]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _dtype_code(X: np.ndarray) -> int:
    if X.dtype == np.uint8:
        return 0
    if X.dtype == np.float32:
        return 1
    raise TypeError(f"oracle supports uint8 / float32 vectors, got {X.dtype}")


def nthreads_default() -> int:
    return os.cpu_count() or 1


class Index:
    """The oracle's view of the label-centric index (Alg. 1)."""

    def __init__(self, X, post_off, post_ids, T, R, graph_off=None, graph_ids=None):
        self.X = np.ascontiguousarray(X)
        self.dtype = _dtype_code(self.X)
        self.N, self.dim = self.X.shape
        self.post_off = np.ascontiguousarray(post_off, dtype=np.int64)
        self.post_ids = np.ascontiguousarray(post_ids, dtype=np.int32)
        self.L = len(self.post_off) - 1
        self.T, self.R = int(T), int(R)
        if graph_off is None:
            graph_off = np.zeros(self.L + 1, dtype=np.int64)
            graph_ids = np.zeros(1, dtype=np.int32)
        self.graph_off = np.ascontiguousarray(graph_off, dtype=np.int64)
        self.graph_ids = np.ascontiguousarray(graph_ids, dtype=np.int32)
        if self.graph_ids.size == 0:
            self.graph_ids = np.zeros(1, dtype=np.int32)
        self._h = lib().or_index_create(self.dtype, self.dim, self.N, _ptr(self.X), self.L,
                                        _ptr(self.post_off), _ptr(self.post_ids), self.T, self.R,
                                        _ptr(self.graph_off), _ptr(self.graph_ids))

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:     # module globals may be gone at exit
            try:
                lib().or_index_free(self._h)
            except TypeError:
                pass
            self._h = None

    def point_labels(self):
        """The predicate table (global label array + per-point offsets)."""
        total = lib().or_index_pt_off(self._h, self.N)
        off = np.array([lib().or_index_pt_off(self._h, i) for i in range(self.N + 1)], np.int64) \
            if self.N <= 200_000 else None
        lab_p = lib().or_index_pt_lab(self._h)
        lab = np.ctypeslib.as_array(C.cast(lab_p, C.POINTER(C.c_int32)), shape=(max(total, 1),))
        return off, lab[:total].copy()

    # -- the method ----------------------------------------------------------------
    def search(self, Q, q_off, q_lab, k=10, itopk=64, op="single", recall_mode="greedy",
               exact=False, search_width=1, n_init=0, max_iterations=0, seed=0x5EED1234,
               forced_entry=-1, nthreads=None, counters=False, max_items_per_q=8, and_scan_threshold=0,
               scan_threshold=0):
        Q = np.ascontiguousarray(Q, dtype=self.X.dtype)
        q_off = np.ascontiguousarray(q_off, dtype=np.int64)
        q_lab = np.ascontiguousarray(q_lab, dtype=np.int32)
        n = len(q_off) - 1
        ids = np.empty((n, k), np.int32)
        d = np.empty((n, k), np.float64)
        ctr = np.full((n, max_items_per_q, 4), -1, np.int64) if counters else None
        rc = lib().or_search(self._h, n, _ptr(Q), _ptr(q_off), _ptr(q_lab), OP[op],
                             RECALL_MODE[recall_mode], int(exact), k, itopk, search_width, n_init,
                             max_iterations, seed & 0xFFFFFFFF, forced_entry, _ptr(ids), _ptr(d),
                             _ptr(ctr) if ctr is not None else None, max_items_per_q,
                             nthreads or nthreads_default(), int(and_scan_threshold), int(scan_threshold))
        if rc != 0:
            raise ValueError("oracle: invalid query (SINGLE with more than one label)")
        return (ids, d, ctr) if counters else (ids, d)

    def label_knn(self, label, K):
        """f4: the K nearest other members of every point of `label` by (squared L2, local id),
        exact (plain sort); [S][K] local ids, -1 padded."""
        S = int(self.post_off[label + 1] - self.post_off[label])
        out = np.empty((S, K), np.int32)
        lib().or_label_knn(self._h, int(label), int(K), _ptr(out))
        return out

    def exact_knn(self, Q, q_off, q_lab, k=10, op="single", nthreads=None):
        """Definition 1 ground truth by brute force over all N points."""
        Q = np.ascontiguousarray(Q, dtype=self.X.dtype)
        q_off = np.ascontiguousarray(q_off, dtype=np.int64)
        q_lab = np.ascontiguousarray(q_lab, dtype=np.int32)
        n = len(q_off) - 1
        ids = np.empty((n, k), np.int32)
        d = np.empty((n, k), np.float64)
        lib().or_exact_knn(self._h, n, _ptr(Q), _ptr(q_off), _ptr(q_lab), OP[op], k, _ptr(ids),
                           _ptr(d), nthreads or nthreads_default())
        return ids, d

    def route(self, q_off, q_lab, op="single", recall_mode="greedy", exact=False, and_scan_threshold=0,
              scan_threshold=0):
        q_off = np.ascontiguousarray(q_off, dtype=np.int64)
        q_lab = np.ascontiguousarray(q_lab, dtype=np.int32)
        n = len(q_off) - 1
        nmax = int(q_off[-1]) + 1
        out = np.empty((nmax, 5), np.int32)
        pred = np.empty(max(1, int(np.sum(np.diff(q_off) ** 2)) + 1), np.int32)
        m = lib().or_route(self._h, n, _ptr(q_off), _ptr(q_lab), OP[op], RECALL_MODE[recall_mode],
                           int(exact), int(and_scan_threshold), int(scan_threshold), _ptr(out), nmax,
                           _ptr(pred))
        if m < 0:
            raise ValueError("oracle: invalid query")
        return out[:m].copy(), pred


def verify(point_labels_sorted, P, trace=False):
    """Boundary-narrowing predicate on one point's sorted label list."""
    a = np.ascontiguousarray(point_labels_sorted, dtype=np.int32)
    p = np.ascontiguousarray(P, dtype=np.int32)
    tr = np.full(3 * max(1, len(p)), -7, np.int64)
    ok = lib().or_verify(_ptr(a) if a.size else None, 0, len(a), _ptr(p) if p.size else None,
                         len(p), _ptr(tr))
    return (bool(ok), tr.reshape(-1, 3)) if trace else bool(ok)


def query_hash(q: np.ndarray) -> int:
    q = np.ascontiguousarray(q)
    return int(lib().or_query_hash(_dtype_code(q.reshape(1, -1)), q.size, _ptr(q)))


def entry_hash(seed: int, qh: int, label: int, i: int, S: int) -> int:
    return int(lib().or_entry_hash(seed & 0xFFFFFFFF, qh & 0xFFFFFFFF, label, i, S))


def cagra_rows(knn, R):
    """f4: CAGRA rank pruning + reverse edges + row assembly (oracle.c or_cagra_rows) on kNN lists
    [S][K] of local ids; returns (pruned [S][R], rows [S][R])."""
    knn = np.ascontiguousarray(knn, np.int32)
    S, K = knn.shape
    pruned = np.empty((S, R), np.int32)
    rows = np.empty((S, R), np.int32)
    lib().or_cagra_rows(S, K, _ptr(knn), int(R), _ptr(pruned), _ptr(rows))
    return pruned, rows


def merge(ids_lists, dists_lists, k):
    """Alg. 2 L431 merge of per-item lists (each of length k, -1 padded)."""
    ids = np.ascontiguousarray(np.asarray(ids_lists, np.int32).reshape(-1))
    d = np.ascontiguousarray(np.asarray(dists_lists, np.float64).reshape(-1))
    n_lists = ids.size // k
    oi = np.empty(k, np.int32)
    od = np.empty(k, np.float64)
    lib().or_merge(n_lists, k, _ptr(ids), _ptr(d), _ptr(oi), _ptr(od))
    return oi, od


def memory_model_gib(N, D, R, Rp, F, F_HS, F_LS, b):
    """P:L497-L500 memory model in GiB: (hs, ls, total, single, mapping)."""
    L = lib()
    g = float(1 << 30)
    hs = L.or_mem_hs_bytes(N, D, F_HS, Rp, b) / g
    ls = L.or_mem_ls_bytes(N, D, F_LS, b) / g
    return hs, ls, hs + ls, L.or_mem_single_bytes(N, D, R, b) / g, L.or_mem_map_bytes(N, F, b) / g


# Recall@K (reading #24) is a measurement over result arrays, not part of the
# method: one definition, shared with bench.py, pinned in tests/test_metrics.py.
from workload.metrics import recall_at_k, recall_per_query  # noqa: E402,F401
