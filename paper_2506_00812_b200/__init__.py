"""Thin Python binding of libvecflow (include/vf.h) -- argument marshalling only.

Every step of the search runs in the library's CUDA kernels; this module converts numpy arrays /
torch tensors into pointers and calls the C-ABI with the same names (vf_build_index, vf_search,
vf_free, ...). There is no CPU fallback: if the extension is missing or no CUDA device is present
the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VF_LIB") or os.path.join(_HERE, "libvecflow.so")   # VF_LIB: A/B builds

VF_OK, VF_ERR_INVALID_ARG, VF_ERR_OUT_OF_MEMORY, VF_ERR_CUDA, VF_ERR_NCCL, VF_ERR_INTERNAL = range(6)
VF_U8, VF_F32 = 0, 1
VF_SINGLE, VF_OR, VF_AND = 0, 1, 2
VF_RECALL_GREEDY, VF_RECALL_PARALLEL = 0, 1
OPS = {"single": VF_SINGLE, "or": VF_OR, "and": VF_AND}
MODES = {"greedy": VF_RECALL_GREEDY, "parallel": VF_RECALL_PARALLEL}
EXPORTED = ("vf_build_index", "vf_search", "vf_free", "vf_last_error", "vf_get_index_info",
            "vf_serve_start", "vf_serve_submit", "vf_serve_wait", "vf_serve_stop", "vf_serve_info",
            "vf_serve_run", "vf_serve_stats",
            "vf_set_profiling", "vf_get_last_stats", "vf_get_last_items", "vf_build_index_virtual_shards",
            "vf_partition_labels", "vf_build_graphs")


class VfError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"vf status {status}: {msg}")
        self.status = status


class BuildDesc(C.Structure):
    _fields_ = [("n_points", C.c_int64), ("dim", C.c_int32), ("dtype", C.c_int32),
                ("vectors", C.c_void_p), ("n_labels", C.c_int32),
                ("posting_offsets", C.c_void_p), ("posting_ids", C.c_void_p),
                ("threshold_T", C.c_int32), ("degree_R", C.c_int32),
                ("graph_row_offsets", C.c_void_p), ("graph_local_ids", C.c_void_p),
                ("world_size", C.c_int32), ("rank", C.c_int32), ("nccl_unique_id", C.c_void_p),
                ("device", C.c_int32)]


class GraphDesc(C.Structure):
    _fields_ = [("n_points", C.c_int64), ("dim", C.c_int32), ("dtype", C.c_int32),
                ("vectors", C.c_void_p), ("n_labels", C.c_int32),
                ("posting_offsets", C.c_void_p), ("posting_ids", C.c_void_p),
                ("threshold_T", C.c_int32), ("degree_R", C.c_int32), ("knn_k", C.c_int32),
                ("exact_max", C.c_int64), ("ivf_cell", C.c_int32), ("ivf_probes", C.c_int32),
                ("kmeans_iters", C.c_int32), ("device", C.c_int32), ("knn_lists", C.c_void_p)]


class GraphReport(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("ms_total", "ms_upload", "ms_knn_exact", "ms_kmeans", "ms_knn_ivf",
                                          "ms_prune", "ms_rows", "ms_download")] + \
               [(n, C.c_int64) for n in ("n_graph_labels", "n_exact_labels", "n_ivf_labels", "rows", "join_pairs")] + \
               [("knn_k", C.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class SearchParams(C.Structure):
    _fields_ = [("k", C.c_int32), ("itopk", C.c_int32), ("search_width", C.c_int32),
                ("n_init", C.c_int32), ("max_iterations", C.c_int32), ("seed", C.c_uint32),
                ("op", C.c_int32), ("recall_mode", C.c_int32), ("exact", C.c_int32),
                ("and_scan_threshold", C.c_int32), ("scan_threshold", C.c_int32), ("n_query_labels", C.c_int64)]


class IndexInfo(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("n_points", "n_labels", "n_hs_labels", "n_ls_labels",
                                         "hs_rows", "ls_rows")] + \
               [("row_bytes", C.c_int32), ("degree_R", C.c_int32)] + \
               [(n, C.c_int64) for n in ("bytes_vectors", "bytes_graph", "bytes_map_hs",
                                         "bytes_ls_vectors", "bytes_map_ls", "bytes_predicate",
                                         "bytes_directory", "bytes_norms", "bytes_u8_store",
                                         "bytes_total")] + \
               [("world_size", C.c_int32), ("rank", C.c_int32), ("owned_labels", C.c_int64)]


class SearchStats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("n_queries", "n_items", "n_scan_items", "n_graph_items",
                                         "n_segments", "n_tiles", "scan_rows", "scan_query_rows",
                                         "graph_V", "graph_E", "graph_iterations", "graph_V_max")] + \
               [(n, C.c_double) for n in ("ms_route", "ms_scan", "ms_graph", "ms_merge", "ms_copy",
                                          "ms_total")] + \
               [("kernel_launches", C.c_int32), ("row_bytes", C.c_int32), ("n_profiled", C.c_int64)] + \
               [(n, C.c_double) for n in ("mean_ms_route", "mean_ms_scan", "mean_ms_graph", "mean_ms_merge",
                                          "mean_ms_copy", "mean_ms_total", "ms_scan_active", "ms_graph_active")] + \
               [("n_invalid_queries", C.c_int64), ("prefilter_words", C.c_int64)] + \
               [("ms_filter", C.c_double), ("mean_ms_filter", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None


def lib():
    """Load the in-tree libvecflow.so (built by build.py / __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libvecflow.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        p, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        L.vf_build_index.restype = C.c_int
        L.vf_build_index.argtypes = [C.POINTER(BuildDesc), C.POINTER(p)]
        L.vf_search.restype = C.c_int
        L.vf_search.argtypes = [p, p, i64, p, p, C.POINTER(SearchParams), p, p, p]
        L.vf_free.restype = None
        L.vf_free.argtypes = [p]
        L.vf_last_error.restype = C.c_char_p
        L.vf_last_error.argtypes = []
        L.vf_get_index_info.restype = C.c_int
        L.vf_get_index_info.argtypes = [p, C.POINTER(IndexInfo)]
        L.vf_set_profiling.restype = C.c_int
        L.vf_set_profiling.argtypes = [p, i32]
        L.vf_get_last_stats.restype = C.c_int
        L.vf_get_last_stats.argtypes = [p, p, C.POINTER(SearchStats)]
        L.vf_get_last_items.restype = C.c_int
        L.vf_get_last_items.argtypes = [p, p, i64, p, C.POINTER(i64)]
        L.vf_serve_start.restype = C.c_int
        L.vf_serve_start.argtypes = [p, C.POINTER(SearchParams), i32, i32, C.POINTER(p)]
        L.vf_serve_submit.restype = C.c_int
        L.vf_serve_submit.argtypes = [p, p, p, i32, C.POINTER(i64)]
        L.vf_serve_wait.restype = C.c_int
        L.vf_serve_wait.argtypes = [p, i64, p, p]
        L.vf_serve_stop.restype = C.c_int
        L.vf_serve_stop.argtypes = [p]
        L.vf_serve_run.restype = C.c_int
        L.vf_serve_run.argtypes = [p, i64, p, p, p, i32, p, p]
        L.vf_serve_stats.restype = C.c_int
        L.vf_serve_stats.argtypes = [p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                     C.POINTER(i64)]
        L.vf_serve_info.restype = C.c_int
        L.vf_serve_info.argtypes = [p, C.POINTER(i32), C.POINTER(i64)]
        L.vf_build_index_virtual_shards.restype = C.c_int
        L.vf_build_index_virtual_shards.argtypes = [C.POINTER(BuildDesc), i32, C.POINTER(p)]
        L.vf_build_graphs.restype = C.c_int
        L.vf_build_graphs.argtypes = [C.POINTER(GraphDesc), p, p, C.POINTER(GraphReport)]
        L.vf_partition_labels.restype = C.c_int
        L.vf_partition_labels.argtypes = [i32, p, i32, p]
        _lib = L
    return _lib


def _check(status):
    if status != VF_OK:
        raise VfError(status, lib().vf_last_error().decode())


def _ptr(x):
    """Pointer of a numpy array or a torch tensor (host or device); None for None."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        return x.ctypes.data_as(C.c_void_p)
    return C.c_void_p(x.data_ptr())


def _dtype_code(X) -> int:
    dt = str(X.dtype)
    if dt in ("uint8", "torch.uint8"):
        return VF_U8
    if dt in ("float32", "torch.float32"):
        return VF_F32
    raise TypeError(f"vectors must be uint8 or float32, got {dt}")


def _stream_ptr(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


class Index:
    """Device-resident label-centric index: vf_build_index / vf_search / vf_free."""

    def __init__(self, X, post_off, post_ids, threshold_T, degree_R=16, graph_off=None,
                 graph_ids=None, device=0, world_size=1, rank=0, nccl_unique_id=None, virtual_shards=0):
        X = np.ascontiguousarray(X)
        self._keep = [X, np.ascontiguousarray(post_off, np.int64), np.ascontiguousarray(post_ids, np.int32)]
        self.dtype = _dtype_code(X)
        self.dim = X.shape[1]
        self.n_labels = len(post_off) - 1
        d = BuildDesc()
        d.n_points, d.dim, d.dtype = X.shape[0], X.shape[1], self.dtype
        d.vectors = _ptr(X)
        d.n_labels = self.n_labels
        d.posting_offsets, d.posting_ids = _ptr(self._keep[1]), _ptr(self._keep[2])
        d.threshold_T, d.degree_R = int(threshold_T), int(degree_R)
        if graph_off is not None:
            go = np.ascontiguousarray(graph_off, np.int64)
            gi = np.ascontiguousarray(graph_ids, np.int32)
            if gi.size == 0:
                gi = np.full(1, -1, np.int32)
            self._keep += [go, gi]
            d.graph_row_offsets, d.graph_local_ids = _ptr(go), _ptr(gi)
        d.world_size, d.rank, d.device = int(world_size), int(rank), int(device)
        if nccl_unique_id is not None:
            self._uid = C.create_string_buffer(bytes(nccl_unique_id), 128)
            d.nccl_unique_id = C.cast(self._uid, C.c_void_p)
        h = C.c_void_p()
        if virtual_shards:
            _check(lib().vf_build_index_virtual_shards(C.byref(d), int(virtual_shards), C.byref(h)))
        else:
            _check(lib().vf_build_index(C.byref(d), C.byref(h)))
        self._h = h
        self._keep = None   # the library copied everything

    def close(self):
        if getattr(self, "_h", None):
            lib().vf_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        i = IndexInfo()
        _check(lib().vf_get_index_info(self._h, C.byref(i)))
        return {f: getattr(i, f) for f, _ in i._fields_}

    def set_profiling(self, enable=True):
        _check(lib().vf_set_profiling(self._h, 1 if enable else 0))

    def search_into(self, Q, q_off, q_lab, out_ids, out_dists, k=10, itopk=64, op="single",
                    recall_mode="greedy", exact=False, search_width=1, n_init=0, max_iterations=0,
                    seed=0x5EED1234, and_scan_threshold=0, stream=None, n_query_labels=0,
                    scan_threshold=0):
        """vf_search with caller-provided buffers (numpy host arrays or torch tensors on either
        side). Asynchronous on `stream` when the outputs are device tensors. With device label
        offsets, `n_query_labels` = q_off[-1] (if the caller knows it) avoids a stream sync."""
        p = SearchParams(int(k), int(itopk), int(search_width), int(n_init), int(max_iterations),
                         int(seed) & 0xFFFFFFFF, OPS[op] if isinstance(op, str) else int(op),
                         MODES[recall_mode] if isinstance(recall_mode, str) else int(recall_mode),
                         1 if exact else 0, int(and_scan_threshold), int(scan_threshold), int(n_query_labels))
        n = int(q_off.shape[0]) - 1
        _check(lib().vf_search(self._h, _ptr(Q), n, _ptr(q_off), _ptr(q_lab), C.byref(p),
                               _ptr(out_ids), _ptr(out_dists), _stream_ptr(stream)))

    def serve(self, k=10, itopk=64, op="single", recall_mode="greedy", exact=False, search_width=1, n_init=0,
              max_iterations=0, seed=0x5EED1234, and_scan_threshold=0, scan_threshold=0, capacity=1024,
              n_workers=0):
        """vf_serve_start: a persistent serving kernel on this index (f1); see Server."""
        p = SearchParams(int(k), int(itopk), int(search_width), int(n_init), int(max_iterations),
                         int(seed) & 0xFFFFFFFF, OPS[op] if isinstance(op, str) else int(op),
                         MODES[recall_mode] if isinstance(recall_mode, str) else int(recall_mode),
                         1 if exact else 0, int(and_scan_threshold), int(scan_threshold), 0)
        h = C.c_void_p()
        _check(lib().vf_serve_start(self._h, C.byref(p), int(capacity), int(n_workers), C.byref(h)))
        return Server(h, k, self)

    def search(self, Q, q_off, q_lab, k=10, **kw):
        """Host convenience wrapper: numpy in, numpy out (blocks)."""
        Q = np.ascontiguousarray(Q)
        q_off = np.ascontiguousarray(q_off, np.int64)
        q_lab = np.ascontiguousarray(q_lab, np.int32)
        if q_lab.size == 0:
            q_lab = np.zeros(1, np.int32)
        n = len(q_off) - 1
        ids = np.empty((n, k), np.int32)
        d = np.empty((n, k), np.float32)
        self.search_into(Q, q_off, q_lab, ids, d, k=k, **kw)
        return ids, d

    def last_stats(self, stream=None) -> dict:
        s = SearchStats()
        _check(lib().vf_get_last_stats(self._h, _stream_ptr(stream), C.byref(s)))
        return s.as_dict()

    def last_items(self, stream=None) -> np.ndarray:
        n = C.c_int64()
        _check(lib().vf_get_last_items(self._h, _stream_ptr(stream), 0, None, C.byref(n)))
        rec = np.empty((max(n.value, 1), 6), np.int32)
        _check(lib().vf_get_last_items(self._h, _stream_ptr(stream), n.value, _ptr(rec), C.byref(n)))
        return rec[:n.value]


class Server:
    """Persistent-kernel serving (vf_serve_*): submit(query, labels) -> ticket; wait(ticket) -> (ids,
    dists). Host numpy in and out; one query per call (the single-batch mode of P:L733)."""

    def __init__(self, h, k, index):
        self._h, self.k, self._index = h, int(k), index

    def submit(self, q, labels) -> int:
        q = np.ascontiguousarray(q)
        lab = np.ascontiguousarray(labels, np.int32).reshape(-1)
        t = C.c_int64()
        _check(lib().vf_serve_submit(self._h, _ptr(q), _ptr(lab) if lab.size else None, int(lab.size),
                                     C.byref(t)))
        return t.value

    def wait(self, ticket, out_ids=None, out_dists=None):
        ids = np.empty(self.k, np.int32) if out_ids is None else out_ids
        d = np.empty(self.k, np.float32) if out_dists is None else out_dists
        _check(lib().vf_serve_wait(self._h, int(ticket), _ptr(ids), _ptr(d)))
        return ids, d

    def run(self, Q, q_off, q_lab, max_in_flight=1024):
        """vf_serve_run: every query of a host batch as its own job (single-batch mode), in C."""
        Q = np.ascontiguousarray(Q)
        q_off = np.ascontiguousarray(q_off, np.int64)
        q_lab = np.ascontiguousarray(q_lab, np.int32)
        if q_lab.size == 0:
            q_lab = np.zeros(1, np.int32)
        n = len(q_off) - 1
        ids = np.empty((n, self.k), np.int32)
        d = np.empty((n, self.k), np.float32)
        _check(lib().vf_serve_run(self._h, n, _ptr(Q), _ptr(q_off), _ptr(q_lab), int(max_in_flight), _ptr(ids),
                                  _ptr(d)))
        return ids, d

    def stats(self) -> dict:
        w, c, s, n = C.c_double(), C.c_double(), C.c_double(), C.c_int64()
        _check(lib().vf_serve_stats(self._h, C.byref(w), C.byref(c), C.byref(s), C.byref(n)))
        return {"wait_us": w.value, "copy_us": c.value, "search_us": s.value, "parts": n.value}

    def info(self) -> dict:
        n, s = C.c_int32(), C.c_int64()
        _check(lib().vf_serve_info(self._h, C.byref(n), C.byref(s)))
        return {"n_workers": n.value, "submitted": s.value}

    def stop(self):
        if self._h:
            h, self._h = self._h, None
            _check(lib().vf_serve_stop(h))

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.stop()

    def __del__(self):
        try:
            self.stop()
        except Exception:
            pass


def partition_labels(sizes, world):
    """vf_partition_labels: label -> rank ownership (greedy LPT over |C_l|)."""
    sizes = np.ascontiguousarray(sizes, np.int64)
    owner = np.empty(max(1, sizes.size), np.int32)
    _check(lib().vf_partition_labels(sizes.size, _ptr(sizes), int(world), _ptr(owner)))
    return owner[:sizes.size]


def nccl_unique_id():
    """A fresh 128-byte ncclUniqueId (rank 0 creates it and broadcasts it with torch.distributed)."""
    import ctypes.util
    h = C.CDLL("libnccl.so.2")
    buf = C.create_string_buffer(128)
    if h.ncclGetUniqueId(buf) != 0:
        raise VfError(VF_ERR_NCCL, "ncclGetUniqueId failed")
    return bytes(buf.raw)


def build_graphs(X, post_off, post_ids, threshold_T, degree_R=16, knn_k=0, exact_max=0, ivf_cell=0, ivf_probes=0,
                 kmeans_iters=0, device=0, return_knn=False):
    """vf_build_graphs (f4): the per-label graphs built on the GPU. Returns (graph_off int64[L+1],
    graph_ids int32[rows*R], report dict[, knn int32[rows][knn_k]])."""
    X = np.ascontiguousarray(X)
    post_off = np.ascontiguousarray(post_off, np.int64)
    post_ids = np.ascontiguousarray(post_ids, np.int32)
    L = len(post_off) - 1
    sizes = np.diff(post_off)
    rows = int(sizes[sizes >= threshold_T].sum())
    goff = np.empty(L + 1, np.int64)
    gids = np.empty(max(rows * degree_R, 1), np.int32)
    kk = knn_k if knn_k > 0 else min(32, 2 * degree_R)
    kk = 16 if kk <= 16 else 32
    knn = np.empty((max(rows, 1), kk), np.int32) if return_knn else None
    d = GraphDesc(X.shape[0], X.shape[1], _dtype_code(X), X.ctypes.data, L, post_off.ctypes.data,
                  post_ids.ctypes.data if post_ids.size else None, int(threshold_T), int(degree_R), int(knn_k),
                  int(exact_max), int(ivf_cell), int(ivf_probes), int(kmeans_iters), int(device),
                  knn.ctypes.data if knn is not None else None)
    rep = GraphReport()
    _check(lib().vf_build_graphs(C.byref(d), goff.ctypes.data, gids.ctypes.data, C.byref(rep)))
    gids = gids[:rows * degree_R]
    if return_knn:
        return goff, gids, rep.as_dict(), knn[:rows]
    return goff, gids, rep.as_dict()
