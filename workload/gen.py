"""Seeded synthetic workload generator (input recipe: DESIGN.md §3).

Shapes follow the paper's workloads (§5.1) and BASELINE.json configs:
  * vectors   -- "clustered low-rank" points, integer valued in [0, 255] (u8 / fp32-int) or the
                 pre-rounding value / 255 (fp32-float, tiny only);
  * labels    -- the semi-synthetic Zipf recipe of PAPER.md L583-L586: label j (0-based) enters
                 point i independently with p_j = c / (j + 1), c = F / H_L  (Zipf exponent s = 1,
                 pinned by the "14,000 points" least-specific SIFT-1M cluster);
  * queries   -- fresh vectors from the same mixture; labels drawn from a uniformly random base
                 point (frequency-weighted, SURVEY §8(c) reading #28). AND2/OR2 take two distinct
                 labels of a base point that has at least two, so |AND set| >= 1.

Everything is drawn from numpy PCG64 streams with fixed seeds (vectors 1001, labels 1002, query
vectors 1003, query labels 1004); vectors in 2^18-row chunks, chunk i from SeedSequence(seed)
spawn i (float32 draws), so a (config, variant) pair always yields bit-identical arrays. No distance, routing, search or merge arithmetic lives here.
"""
from __future__ import annotations

import dataclasses
import math
import os

import numpy as np

SEED_VECTORS = 1001
SEED_LABELS = 1002
SEED_QVECTORS = 1003
SEED_QLABELS = 1004
SEARCH_SEED = 0x5EED1234

_CHUNK = 1 << 18  # rows per generation chunk (part of the recipe: changing it changes the data)


@dataclasses.dataclass
class VectorModel:
    """Parameters of the clustered low-rank (CLR) vector model."""
    rank: int          # latent dimension r
    clusters: int      # mixture components C
    center_scale: float = 1.5   # latent cluster centres m_c ~ N(0, center_scale^2 I_r)
    sigma_x: float = 40.0       # per-coordinate std of the projected signal
    sigma_n: float = 3.0        # iid per-coordinate noise


@dataclasses.dataclass
class Config:
    name: str
    n_points: int
    dim: int
    n_labels: int
    mean_labels: float      # F
    threshold_T: int
    n_queries: int
    query_mode: str         # "single" | "and2" | "or2" | "mix_and" (50% single / 50% and2)
    k: int
    degree_R: int
    model: VectorModel
    dtype: str              # "u8" | "f32int" | "f32float"


CONFIGS = {
    # BASELINE.json configs[0]
    "tiny": Config("tiny", 10_000, 32, 50, 3.17, 1000, 1000, "single", 10, 16,
                   VectorModel(rank=8, clusters=16), "f32int"),
    # BASELINE.json configs[1]
    "sift": Config("sift", 1_000_000, 128, 1000, 3.17, 2000, 10_000, "single", 10, 16,
                   VectorModel(rank=12, clusters=256), "f32int"),
    # BASELINE.json configs[2]
    "yfcc": Config("yfcc", 10_000_000, 192, 200_386, 10.8, 2000, 100_000, "mix_and", 10, 16,
                   VectorModel(rank=16, clusters=1024), "u8"),
}


def config(name: str, **overrides) -> Config:
    c = dataclasses.replace(CONFIGS[name])
    for k, v in overrides.items():
        setattr(c, k, v)
    return c


# ----------------------------------------------------------------------------- vectors
def _clr_chunk(seq: np.random.SeedSequence, n: int, dim: int, m: VectorModel, A: np.ndarray,
               centers: np.ndarray, dtype: str) -> np.ndarray:
    """n points of the CLR model, 128 + A z + sigma_n * eps, finished to the storage dtype."""
    rng = np.random.Generator(np.random.PCG64(seq))
    c = rng.integers(0, m.clusters, size=n)
    z = centers[c] + rng.standard_normal((n, m.rank), dtype=np.float32)
    x = z @ A.T
    x += rng.standard_normal((n, dim), dtype=np.float32) * np.float32(m.sigma_n)
    x += np.float32(128.0)
    if dtype == "f32float":
        return x / np.float32(255.0)
    np.rint(x, out=x)
    np.clip(x, 0, 255, out=x)
    if dtype == "u8":
        return x.astype(np.uint8)
    if dtype == "f32int":
        return x
    raise ValueError(dtype)


def _model_params(dim: int, m: VectorModel):
    rng = np.random.Generator(np.random.PCG64(SEED_VECTORS + 7919))
    scale = m.sigma_x / math.sqrt(m.rank * (1.0 + m.center_scale ** 2))
    A = (rng.standard_normal((dim, m.rank)) * scale).astype(np.float32)
    centers = (rng.standard_normal((m.clusters, m.rank)) * m.center_scale).astype(np.float32)
    return A, centers


def _clr(cfg: Config, n: int, seed: int) -> np.ndarray:
    """Chunk i of 2^18 rows draws from its own stream SeedSequence(seed).spawn()[i], so the result
    does not depend on how many threads generate it."""
    from concurrent.futures import ThreadPoolExecutor
    A, centers = _model_params(cfg.dim, cfg.model)
    n_chunks = (n + _CHUNK - 1) // _CHUNK
    seqs = np.random.SeedSequence(seed).spawn(max(n_chunks, 1))
    out = np.empty((n, cfg.dim), dtype=np.uint8 if cfg.dtype == "u8" else np.float32)

    def work(i):
        s0, e0 = i * _CHUNK, min(n, (i + 1) * _CHUNK)
        out[s0:e0] = _clr_chunk(seqs[i], e0 - s0, cfg.dim, cfg.model, A, centers, cfg.dtype)

    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as ex:
        list(ex.map(work, range(n_chunks)))
    return out


def gen_vectors(cfg: Config, seed: int = SEED_VECTORS) -> np.ndarray:
    return _clr(cfg, cfg.n_points, seed)


def gen_query_vectors(cfg: Config, n: int | None = None, seed: int = SEED_QVECTORS) -> np.ndarray:
    return _clr(cfg, cfg.n_queries if n is None else n, seed)


# ----------------------------------------------------------------------------- labels
def zipf_probabilities(n_labels: int, mean_labels: float) -> np.ndarray:
    """p_j = c / (j+1), c = F / H_L (s = 1)."""
    H = np.sum(1.0 / np.arange(1, n_labels + 1, dtype=np.float64))
    c = mean_labels / H
    return c / np.arange(1, n_labels + 1, dtype=np.float64)


def gen_postings(cfg: Config, seed: int = SEED_LABELS):
    """Posting lists C_l as CSR: offsets int64[L+1], ids int32 (ascending per list).

    Each label j is an independent Bernoulli(p_j) draw per point. Zero-label points are allowed
    (SURVEY reading #27)."""
    N, L = cfg.n_points, cfg.n_labels
    p = zipf_probabilities(L, cfg.mean_labels)
    rng = np.random.Generator(np.random.PCG64(seed))
    lists = []
    for j in range(L):
        if p[j] >= 0.05:
            ids = np.flatnonzero(rng.random(N) < p[j]).astype(np.int32)
        else:
            nj = int(rng.binomial(N, p[j]))
            ids = np.sort(rng.choice(N, size=nj, replace=False)).astype(np.int32)
        lists.append(ids)
    sizes = np.array([len(a) for a in lists], dtype=np.int64)
    offsets = np.zeros(L + 1, dtype=np.int64)
    np.cumsum(sizes, out=offsets[1:])
    ids = np.concatenate(lists).astype(np.int32) if lists else np.zeros(0, np.int32)
    return offsets, ids


def point_labels(n_points: int, offsets: np.ndarray, ids: np.ndarray):
    """Transpose of the posting CSR: per-point sorted label lists (generator bookkeeping)."""
    lab = np.repeat(np.arange(len(offsets) - 1, dtype=np.int32), np.diff(offsets))
    order = np.lexsort((lab, ids))
    cnt = np.bincount(ids, minlength=n_points).astype(np.int64)
    poff = np.zeros(n_points + 1, dtype=np.int64)
    np.cumsum(cnt, out=poff[1:])
    return poff, lab[order].astype(np.int32)


# ----------------------------------------------------------------------------- queries
def gen_query_labels(cfg: Config, offsets: np.ndarray, ids: np.ndarray,
                     n: int | None = None, mode: str | None = None, seed: int = SEED_QLABELS):
    """Query label CSR (qoff int64[n+1], qlab int32). Labels of a uniformly random base point."""
    n = cfg.n_queries if n is None else n
    mode = cfg.query_mode if mode is None else mode
    poff, plab = point_labels(cfg.n_points, offsets, ids)
    cnt = np.diff(poff)
    rng = np.random.Generator(np.random.PCG64(seed))
    one = np.flatnonzero(cnt >= 1)
    two = np.flatnonzero(cnt >= 2)
    if mode == "single":
        want2 = np.zeros(n, dtype=bool)
    elif mode in ("and2", "or2"):
        want2 = np.ones(n, dtype=bool)
    elif mode == "mix_and":
        want2 = rng.random(n) < 0.5
    else:
        raise ValueError(mode)
    u0 = rng.random(n)
    u1 = rng.random(n)
    u2 = rng.random(n)
    qoff = np.zeros(n + 1, dtype=np.int64)
    qoff[1:] = np.cumsum(np.where(want2, 2, 1))
    qlab = np.empty(int(qoff[-1]), dtype=np.int32)
    for i in range(n):
        if want2[i]:
            b = two[min(int(u0[i] * len(two)), len(two) - 1)]
            c = int(cnt[b])
            i1 = min(int(u1[i] * c), c - 1)
            i2 = min(int(u2[i] * (c - 1)), c - 2)
            if i2 >= i1:
                i2 += 1
            qlab[qoff[i]] = plab[poff[b] + i1]
            qlab[qoff[i] + 1] = plab[poff[b] + i2]
        else:
            b = one[min(int(u0[i] * len(one)), len(one) - 1)]
            c = int(cnt[b])
            qlab[qoff[i]] = plab[poff[b] + min(int(u1[i] * c), c - 1)]
    return qoff, qlab


@dataclasses.dataclass
class Workload:
    cfg: Config
    X: np.ndarray            # [N, D] u8 or f32
    post_off: np.ndarray     # int64 [L+1]
    post_ids: np.ndarray     # int32
    Q: np.ndarray            # [n, D]
    q_off: np.ndarray        # int64 [n+1]
    q_lab: np.ndarray        # int32


def make_workload(name: str, n_queries: int | None = None, query_mode: str | None = None,
                  query_stream: int = 0, **overrides) -> Workload:
    """query_stream > 0 draws an independent query batch (seeds + 7 * query_stream), e.g. one per
    rank of a weak-scaling run; the index data do not change."""
    cfg = config(name, **overrides)
    if n_queries is not None:
        cfg.n_queries = n_queries
    if query_mode is not None:
        cfg.query_mode = query_mode
    X = gen_vectors(cfg)
    off, ids = gen_postings(cfg)
    Q = gen_query_vectors(cfg, seed=SEED_QVECTORS + 7 * query_stream)
    qoff, qlab = gen_query_labels(cfg, off, ids, seed=SEED_QLABELS + 7 * query_stream)
    return Workload(cfg, X, off, ids, Q, qoff, qlab)
