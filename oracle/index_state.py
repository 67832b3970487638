"""Oracle: index state, distance, bucket partition/lookup, append, GRAB container.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). CPU restatement of the
reference's storage layer; every function cites the reference file:line whose
behaviour it restates (paths relative to /root/reference/pkg/src/bucketann).

numpy 2.3.5 semantics matter here: Python-float bounds compared against f32
arrays are rounded to f32 first (NEP 50), which is what the CUDA kernels do
with ``__double2float_rn``.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

SENTINEL = np.uint32(0xFFFFFFFF)  # layout.py:19


class CapacityError(RuntimeError):  # core.py:21
    pass


class DimensionMismatchError(ValueError):  # core.py:17
    pass


@dataclass(frozen=True)
class BuildCfg:
    """BuildParams defaults (core.py:85-118)."""

    k_max: int = 32
    k_local: int = 16
    bucket_capacity: int = 10_000
    proximal_fraction: float = 0.5
    proximal_window: float = 0.2
    alpha: float = 0.6
    rng_seed: int = 0

    @property
    def k_remote(self) -> int:
        return self.k_max - self.k_local


@dataclass(frozen=True)
class SearchCfg:
    """SearchParams defaults (core.py:121-147); range held as (lower, upper)."""

    k: int = 10
    lower: float = -np.inf
    upper: float = np.inf
    itopk: int = 128
    search_width: int = 4
    max_iterations: int = 50
    seed_count: int | None = None
    rng_seed: int = 0

    @property
    def want(self) -> int:  # core.py:142-147
        return self.seed_count if self.seed_count is not None else min(self.itopk, 32)


def sqdist(q, rows) -> np.ndarray:
    """f64-upcast squared L2 of q against each row (core.py:25-38)."""
    q = np.asarray(q)
    rows = np.asarray(rows)
    if rows.ndim != 2 or q.ndim != 1 or rows.shape[1] != q.shape[0]:
        raise DimensionMismatchError(f"query {q.shape} vs rows {rows.shape}")
    delta = rows.astype(np.float64) - q.astype(np.float64)
    return np.einsum("ij,ij->i", delta, delta)


@dataclass
class OracleIndex:
    """GraphIndex + VectorStore + BucketMeta flattened (layout.py:22-104,226-257)."""

    X: np.ndarray  # f32 [N_cap, d]
    scalars: np.ndarray  # f32 [N_cap]
    ids: np.ndarray  # i64 [N_cap]
    count: int
    adjacency: np.ndarray  # u32 [N_cap, k_max]
    cfg: BuildCfg
    boundaries: np.ndarray | None = None  # f32 [m+1]
    i2b: np.ndarray | None = None  # i32 [N_cap]
    b2i: list[list[int]] = field(default_factory=list)

    @property
    def capacity(self) -> int:
        return self.X.shape[0]

    @property
    def dim(self) -> int:
        return self.X.shape[1]

    @property
    def m(self) -> int:
        return len(self.boundaries) - 1

    @property
    def span(self) -> float:  # layout.py:102-104
        return float(self.boundaries[-1]) - float(self.boundaries[0])


def empty_index(dim: int, capacity: int, cfg: BuildCfg) -> OracleIndex:
    """create_index (layout.py:250-257, 177-178)."""
    return OracleIndex(
        X=np.zeros((capacity, dim), dtype="<f4"),
        scalars=np.zeros(capacity, dtype="<f4"),
        ids=np.full(capacity, -1, dtype="<i8"),
        count=0,
        adjacency=np.full((capacity, cfg.k_max), SENTINEL, dtype="<u4"),
        cfg=cfg,
    )


def bucket_lookup(boundaries: np.ndarray, s) -> np.ndarray:
    """bucket_ids_of: f32 searchsorted over interior edges, 'right' (layout.py:157-160)."""
    return np.searchsorted(boundaries[1:-1], np.asarray(s, dtype=np.float32), side="right").astype(np.int32)


def bucket_interval(boundaries: np.ndarray, lower: float, upper: float) -> tuple[int, int]:
    """intersecting_buckets (layout.py:163-174)."""
    lo = int(bucket_lookup(boundaries, np.array([lower], dtype=np.float32))[0])
    hi = int(bucket_lookup(boundaries, np.array([upper], dtype=np.float32))[0])
    return lo, hi


def partition_edges(scalars: np.ndarray, target: int, strategy: str = "quantile") -> np.ndarray:
    """Boundary derivation of partition_buckets (layout.py:107-141)."""
    s = np.asarray(scalars, dtype=np.float32)
    n = len(s)
    if n < 1:
        raise ValueError("cannot partition an empty scalar set")
    if target < 1:
        raise ValueError("target_capacity must be >= 1")
    m = -(-n // target)
    if strategy == "quantile":
        ranks = np.round(np.arange(m + 1) * (n / m)).astype(np.int64)
        ranks[-1] = n - 1
        edges = np.sort(s)[np.minimum(ranks, n - 1)]
    elif strategy == "width":
        edges = np.linspace(s.min(), s.max(), m + 1, dtype=np.float64).astype(np.float32)
        edges[-1] = s.max()
    else:
        raise ValueError(f"unknown bucket strategy: {strategy!r}")
    edges = np.unique(edges).astype("<f4")
    if len(edges) < 2:
        edges = np.array([edges[0], edges[0]], dtype="<f4")
    return edges


def assign_partition(index: OracleIndex, scalars: np.ndarray, strategy: str = "quantile") -> None:
    """partition_buckets map population (layout.py:143-154)."""
    s = np.asarray(scalars, dtype=np.float32)
    index.boundaries = partition_edges(s, index.cfg.bucket_capacity, strategy)
    index.i2b = np.full(index.capacity, -1, dtype="<i4")
    bids = bucket_lookup(index.boundaries, s)
    index.i2b[: len(s)] = bids
    index.b2i = [[] for _ in range(index.m)]
    for slot, b in enumerate(bids.tolist()):
        index.b2i[b].append(slot)


def append_rows(index: OracleIndex, vectors, scalars, ids=None, with_meta: bool = True) -> tuple[int, int]:
    """append_batch (layout.py:181-223): tail claim, row writes, map update."""
    v = np.asarray(vectors, dtype=np.float32)
    s = np.asarray(scalars, dtype=np.float32)
    b = len(v)
    if b == 0:
        return index.count, index.count
    if v.ndim != 2 or v.shape[1] != index.dim:
        raise DimensionMismatchError(f"vectors have shape {v.shape}, index dimension is {index.dim}")
    if len(s) != b:
        raise ValueError(f"{b} vectors but {len(s)} scalars")
    if not np.all(np.isfinite(s)):
        raise ValueError("scalars must be finite")
    start = index.count
    if start + b > index.capacity:
        raise CapacityError(f"capacity exhausted: {start} claimed + {b} requested > {index.capacity}")
    end = start + b
    index.X[start:end] = v
    index.scalars[start:end] = s
    index.ids[start:end] = np.arange(start, end) if ids is None else np.asarray(ids, dtype=np.int64)
    if with_meta and index.boundaries is not None:
        bids = bucket_lookup(index.boundaries, s)
        index.i2b[start:end] = bids
        for off, bid in enumerate(bids.tolist()):
            index.b2i[bid].append(start + off)
    index.count = end
    return start, end


# ---- GRAB v1 container (dataio.py:111-187) --------------------------------
_HDR = struct.Struct("<4sIQQIIIIB")


def container_bytes(index: OracleIndex) -> bytes:
    """save_index byte image (dataio.py:114-139)."""
    n = index.count
    hdr = _HDR.pack(b"GRAB", 1, n, index.capacity, index.dim, index.cfg.k_max,
                    index.cfg.k_local, index.m, 0)
    parts = [
        hdr,
        index.X[:n].astype("<f4").tobytes(),
        index.scalars[:n].astype("<f4").tobytes(),
        index.adjacency[:n].astype("<u4").tobytes(),
        index.boundaries.astype("<f4").tobytes(),
        index.i2b[:n].astype("<u4").tobytes(),
    ]
    return b"".join(parts)


def index_from_container(raw: bytes, cfg: BuildCfg | None = None) -> OracleIndex:
    """load_index (dataio.py:142-187); M_B2I rebuilt in slot order."""
    if raw[:4] != b"GRAB":
        raise ValueError("not an index container")
    _, ver, n, n_cap, d, k_max, k_local, m, metric = _HDR.unpack_from(raw, 0)
    if ver != 1:
        raise ValueError(f"unsupported container version {ver}")
    if metric != 0:
        raise ValueError(f"unsupported metric code {metric}")
    cur = _HDR.size
    chunks = []
    for dt, cnt in (("<f4", n * d), ("<f4", n), ("<u4", n * k_max), ("<f4", m + 1), ("<u4", n)):
        a = np.frombuffer(raw, dtype=dt, count=cnt, offset=cur).copy()
        cur += a.nbytes
        chunks.append(a)
    cfg = cfg or BuildCfg(k_max=k_max, k_local=k_local)
    idx = empty_index(d, n_cap, cfg)
    idx.X[:n] = chunks[0].reshape(n, d)
    idx.scalars[:n] = chunks[1]
    idx.ids[:n] = np.arange(n)
    idx.count = n
    idx.adjacency[:n] = chunks[2].reshape(n, k_max)
    idx.boundaries = chunks[3]
    idx.i2b = np.full(n_cap, -1, dtype="<i4")
    idx.i2b[:n] = chunks[4].astype("<i4")
    idx.b2i = [[] for _ in range(m)]
    for slot, b in enumerate(idx.i2b[:n].tolist()):
        idx.b2i[b].append(slot)
    return idx


def gen_synthetic(n: int, d: int, distribution: str = "gaussian", rng_seed: int = 0,
                  n_clusters: int = 64, cluster_scale: float = 1.5):
    """dataio.py:81-108 draw order (vectors, then scalars)."""
    g = np.random.default_rng(rng_seed)
    if distribution == "gaussian":
        v = g.standard_normal((n, d), dtype=np.float32)
    elif distribution == "clusters":
        c = g.standard_normal((n_clusters, d)).astype(np.float32) * cluster_scale
        a = g.integers(0, n_clusters, size=n)
        v = c[a] + g.standard_normal((n, d), dtype=np.float32)
    else:
        raise ValueError(distribution)
    return v, g.random(n, dtype=np.float32)


def gen_lowrank(n: int, d: int, seed: int, rank: int = 16, noise: float = 0.05, with_scalars: bool = True):
    """SURVEY §8(d) low-rank generator (the data on which R@10 >= 0.95 is reachable)."""
    g = np.random.default_rng(seed)
    W = (g.standard_normal((rank, d)) / 4).astype(np.float32)
    Z = g.standard_normal((n, rank)).astype(np.float32)
    E = g.standard_normal((n, d)).astype(np.float32)
    X = (Z @ W + np.float32(noise) * E).astype(np.float32)
    S = g.random(n, dtype=np.float32) if with_scalars else None
    return X, S


def lowrank_queries(nq: int, d: int, seed: int = 1, rank: int = 16, noise: float = 0.05):
    """Queries from the same low-rank family: W from seed 0, (Z, E) from ``seed``."""
    W = (np.random.default_rng(0).standard_normal((rank, d)) / 4).astype(np.float32)
    g = np.random.default_rng(seed)
    Z = g.standard_normal((nq, rank)).astype(np.float32)
    E = g.standard_normal((nq, d)).astype(np.float32)
    return (Z @ W + np.float32(noise) * E).astype(np.float32)
