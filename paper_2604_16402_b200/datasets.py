"""Synthetic inputs and evaluation helpers used by bench.py and the examples.

* ``gen_synthetic``   reference draw order (dataio.py:81-108)
* ``gen_lowrank`` / ``lowrank_queries``  SURVEY §8(d) low-rank-16 family, the
  data on which R@10 >= 0.95 is reachable at d = 128 (gaussian-128 caps at
  0.895, clusters-128 is disconnected)
* ``generate_ranges`` fixed-width windows (evaluate.py:122-135)
* ``recall_at_k``     evaluate.py:47-57
These are host-side numpy data generators, not part of the GPU compute path.
"""
from __future__ import annotations

import numpy as np

from .params import RangePredicate


def gen_synthetic(n: int, d: int, distribution: str = "gaussian", rng_seed: int = 0, n_clusters: int = 64,
                  cluster_scale: float = 1.5):
    if n < 1 or d < 1:
        raise ValueError("n and d must be >= 1")
    g = np.random.default_rng(rng_seed)
    if distribution == "gaussian":
        v = g.standard_normal((n, d), dtype=np.float32)
    elif distribution == "clusters":
        centers = g.standard_normal((n_clusters, d)).astype(np.float32) * cluster_scale
        v = centers[g.integers(0, n_clusters, size=n)] + g.standard_normal((n, d), dtype=np.float32)
    else:
        raise ValueError(f"unknown distribution: {distribution!r}")
    return v, g.random(n, dtype=np.float32)


def gen_lowrank(n: int, d: int, seed: int = 0, rank: int = 16, noise: float = 0.05, w_seed: int | None = None):
    """``w_seed`` (sharded data): draw the rank-16 basis from default_rng(w_seed)
    and only the coefficients / noise / scalars from ``seed``, so every shard
    shares the query distribution's subspace (lowrank_queries uses seed 0)."""
    g = np.random.default_rng(seed)
    if w_seed is None:
        W = (g.standard_normal((rank, d)) / 4).astype(np.float32)
    else:
        W = (np.random.default_rng(w_seed).standard_normal((rank, d)) / 4).astype(np.float32)
    Z = g.standard_normal((n, rank)).astype(np.float32)
    E = g.standard_normal((n, d)).astype(np.float32)
    X = (Z @ W + np.float32(noise) * E).astype(np.float32)
    return X, g.random(n, dtype=np.float32)


def lowrank_queries(nq: int, d: int, seed: int = 1, rank: int = 16, noise: float = 0.05):
    W = (np.random.default_rng(0).standard_normal((rank, d)) / 4).astype(np.float32)
    g = np.random.default_rng(seed)
    Z = g.standard_normal((nq, rank)).astype(np.float32)
    E = g.standard_normal((nq, d)).astype(np.float32)
    return (Z @ W + np.float32(noise) * E).astype(np.float32)


def generate_ranges(scalars, selectivity: float, n_queries: int, rng_seed: int) -> list[RangePredicate]:
    lo, hi = float(np.min(scalars)), float(np.max(scalars))
    width = selectivity * (hi - lo)
    g = np.random.default_rng([rng_seed, 3, int(round(selectivity * 1_000_000))])
    starts = lo + g.random(n_queries) * ((hi - lo) - width)
    return [RangePredicate(float(s), float(s + width)) for s in starts]


def range_arrays(ranges) -> tuple[np.ndarray, np.ndarray]:
    return (np.array([r.lower for r in ranges], dtype=np.float64),
            np.array([r.upper for r in ranges], dtype=np.float64))


def recall_at_k(result_slots, truth_slots, k: int) -> float:
    truth = {int(s) for s in truth_slots}
    if not truth:
        return float("nan")
    return sum(1 for s in result_slots if int(s) in truth) / min(k, len(truth))


def batch_recall(slots: np.ndarray, counts: np.ndarray, truth: np.ndarray, tcounts: np.ndarray, k: int) -> float:
    vals = [recall_at_k(slots[i, : counts[i]], truth[i, : tcounts[i]], k) for i in range(len(counts))]
    return float(np.nanmean(vals))
