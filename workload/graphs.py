"""Fixture builder for the per-label fixed-degree graphs G_l (test/bench tooling, not the hot path).

The graphs are an INPUT to vf_build_index ("host-built posting lists and per-label graphs",
BASELINE.json north_star); the paper builds them with CAGRA (NN-descent + rank-based reordering,
PAPER.md L348, Alg. 1), which is out of scope. This module builds a
CAGRA-like degree-R graph per HS label from exact k-nearest-neighbour lists:

  knn[j]  = the min(R, S-1) nearest other members of the label, key (d, j') ascending
  row[j]  = knn[j][:R/2]                                   (forward edges)
          + up to R/2 reverse edges u with j in knn[u][:R/2], nearest first
          + knn[j][R/2:] to fill, de-duplicated, padded with -1

Local ids are positions in the ascending posting list C_l. The oracle and the GPU path
consume the same arrays, so the builder's own arithmetic never affects parity.
"""
from __future__ import annotations

import numpy as np


def _knn_numpy(Xl: np.ndarray, K: int) -> np.ndarray:
    S = Xl.shape[0]
    Xd = Xl.astype(np.float64)
    nrm = (Xd * Xd).sum(1)
    out = np.full((S, K), -1, np.int64)
    step = max(1, min(S, (1 << 24) // max(S, 1)))
    for s in range(0, S, step):
        e = min(S, s + step)
        d = nrm[s:e, None] + nrm[None, :] - 2.0 * (Xd[s:e] @ Xd.T)
        d[np.arange(e - s), np.arange(s, e)] = np.inf
        kk = min(K, S - 1)
        if kk <= 0:
            continue
        part = np.argpartition(d, kk - 1, axis=1)[:, :kk] if kk < S else \
            np.tile(np.arange(S), (e - s, 1))
        dp = np.take_along_axis(d, part, axis=1)
        order = np.lexsort((part, dp), axis=1)[:, :kk]   # (d, j) ascending
        out[s:e, :kk] = np.take_along_axis(part, order, axis=1)
    return out


def _knn_torch(Xl: np.ndarray, K: int, device) -> np.ndarray:
    import torch
    S = Xl.shape[0]
    X = torch.from_numpy(np.ascontiguousarray(Xl, dtype=np.float32)).to(device)
    nrm = (X * X).sum(1)
    kk = min(K, S - 1)
    out = np.full((S, K), -1, np.int64)
    if kk <= 0:
        return out
    step = max(256, min(8192, (1 << 28) // max(S, 1)))
    res = []
    for s in range(0, S, step):
        e = min(S, s + step)
        d = nrm[s:e, None] + nrm[None, :] - 2.0 * (X[s:e] @ X.T)
        d[torch.arange(e - s, device=device), torch.arange(s, e, device=device)] = float("inf")
        _, idx = torch.topk(d, kk, dim=1, largest=False, sorted=True)
        res.append(idx.cpu())
    out[:, :kk] = torch.cat(res).numpy()
    return out


def assemble_rows(knn: np.ndarray, R: int) -> np.ndarray:
    """Forward half + reverse edges + fill (see module docstring). knn: [S, R] (-1 padded)."""
    S = knn.shape[0]
    h = R // 2
    fwd = knn[:, :h]
    rest = knn[:, h:R]
    # reverse edges: u -> v for v in fwd[u]; for each v keep the first h sources by rank of v in
    # u's list, then u (a proxy for "nearest first" that needs no distances)
    u = np.repeat(np.arange(S), h)
    rank = np.tile(np.arange(h), S)
    v = fwd.reshape(-1)
    ok = v >= 0
    u, v, rank = u[ok], v[ok], rank[ok]
    order = np.lexsort((u, rank, v))
    u, v = u[order], v[order]
    start = np.searchsorted(v, np.arange(S))
    pos = np.arange(len(v)) - start[v]
    keep = pos < h
    rev = np.full((S, h), -1, np.int64)
    rev[v[keep], pos[keep]] = u[keep]
    cand = np.concatenate([fwd, rev, rest], axis=1)
    valid = cand >= 0
    ncol = cand.shape[1]
    for c in range(1, ncol):
        dup = np.zeros(S, dtype=bool)
        for c2 in range(c):
            dup |= cand[:, c2] == cand[:, c]
        valid[:, c] &= ~dup
    rank = np.cumsum(valid, axis=1) - 1
    sel = valid & (rank < R)
    rows = np.full((S, R), -1, np.int32)
    ri, ci = np.nonzero(sel)
    rows[ri, rank[ri, ci]] = cand[ri, ci]
    return rows


def build_label_graph(Xl: np.ndarray, R: int, device=None) -> np.ndarray:
    S = Xl.shape[0]
    if device is not None and S > 4096:
        knn = _knn_torch(Xl, R, device)
    else:
        knn = _knn_numpy(Xl, R)
    return assemble_rows(knn, R)


def build_graphs(X: np.ndarray, post_off: np.ndarray, post_ids: np.ndarray, T: int, R: int,
                 device=None, labels=None):
    """Graphs for every label with |C_l| >= T (the HS labels).

    Returns (graph_off int64[L+1], graph_ids int32[rows*R]) where rows(l) = |C_l| for HS labels
    and 0 otherwise -- the layout vf_build_index and the oracle both take."""
    L = len(post_off) - 1
    sizes = np.diff(post_off)
    rows_per = np.where(sizes >= T, sizes, 0)
    graph_off = np.zeros(L + 1, np.int64)
    np.cumsum(rows_per, out=graph_off[1:])
    graph_ids = np.full(int(graph_off[-1]) * R, -1, np.int32)
    for l in range(L):
        if rows_per[l] == 0 or (labels is not None and l not in labels):
            continue
        ids = post_ids[post_off[l]:post_off[l + 1]]
        g = build_label_graph(X[ids], R, device)
        graph_ids[graph_off[l] * R:graph_off[l + 1] * R] = g.reshape(-1)
    return graph_off, graph_ids
