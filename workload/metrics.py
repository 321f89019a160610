"""Recall@K -- the measurement definition shared by bench.py and the oracle tests.

Recall@K = |A ∩ GT| / K per query, averaged over queries (Definition of
Recall@K in §2.1). Readings:
  * the denominator is min(K, |GT|): a query whose filter admits fewer than K points is
    scored against all of them; queries whose filter admits none are skipped;
  * GT rows and returned rows are padded with id -1 (ignored);
  * tie-aware variant: a returned id that is not in GT but whose exact distance equals the
    K-th (last) GT distance also counts as a hit -- with ties at the cut-off several answers
    are exact; the score is capped at 1.

This is a metric over already-computed id/distance arrays: it holds none of the search's
arithmetic, so both the oracle's tests and the bench may use it. Pinned by
closed-form cases in tests/test_metrics.py.
"""
from __future__ import annotations

import numpy as np


def recall_per_query(ids, gt_ids, dists=None, gt_dists=None, k=10):
    """Per-query (strict, tie_aware, valid) arrays. `dists` are the returned rows' exact
    distances (same shape as ids) and `gt_dists` the GT distances; without them tie_aware is
    None. `valid` marks queries with a non-empty GT (the others are excluded from means)."""
    ids = np.asarray(ids)[:, :k]
    gt = np.asarray(gt_ids)[:, :k]
    if ids.shape[0] != gt.shape[0]:
        raise ValueError("ids and gt_ids must have the same number of rows")
    gvalid = gt >= 0
    ng = gvalid.sum(axis=1)                               # |GT| (<= K)
    avalid = ids >= 0
    # hits: returned (valid) ids present among the valid GT ids of the same row; a returned row
    # holds distinct ids (a5 dedup), so counting matches per returned entry counts |A ∩ GT|
    eq = (ids[:, :, None] == gt[:, None, :]) & gvalid[:, None, :] & avalid[:, :, None]
    in_gt = eq.any(axis=2)
    hits = in_gt.sum(axis=1)
    den = np.minimum(k, ng)
    valid = ng > 0
    with np.errstate(invalid="ignore", divide="ignore"):
        strict = np.where(valid, hits / np.maximum(den, 1), np.nan)
    tie = None
    if dists is not None and gt_dists is not None:
        d = np.asarray(dists)[:, :k]
        gd = np.asarray(gt_dists)[:, :k]
        rows = np.arange(gt.shape[0])
        kth = gd[rows, np.maximum(ng - 1, 0)]            # the last valid GT distance
        extra = (avalid & ~in_gt & (d == kth[:, None])).sum(axis=1)
        with np.errstate(invalid="ignore", divide="ignore"):
            tie = np.where(valid, np.minimum(1.0, (hits + extra) / np.maximum(den, 1)), np.nan)
    return strict, tie, valid


def recall_at_k(ids, gt_ids, gt_dists=None, dists_exact=None, k=10):
    """Mean recall@K over queries with a non-empty GT: (strict, tie_aware or None).
    `dists_exact` = exact distance of every returned id (enables the tie-aware variant)."""
    s, t, v = recall_per_query(ids, gt_ids, dists_exact, gt_dists, k)
    if not v.any():
        return 1.0, (1.0 if t is not None else None)
    return float(np.mean(s[v])), (float(np.mean(t[v])) if t is not None else None)
