"""``bucketann.layout`` surface (reference layout.py:1-257).

Two kinds of store meet here:

* ``VectorStore(capacity, dim)`` -- the reference's host-side append-only
  store (layout.py:22-79): numpy rows, a lock-serialised contiguous ``claim``
  and a ``publish`` that advances ``count`` only over contiguous completed
  ranges. It is the staging container the phase-level builder helpers
  (``builder.build_local_phase`` / ``build_global_graph``) and the pruning
  primitives take; every computation on it runs in libgrab (rows are uploaded).
* the device index (``GraphIndex``, graph.py): rows live in HBM in bucket slabs;
  ``index.store`` is a read-only reference-shaped view of them.

``append_batch`` serves both: a host ``VectorStore`` is written in place (bucket
ids from the device lookup), a device index appends on the device
(``grab_append``, layout.cu).
"""
from __future__ import annotations

import threading

import numpy as np

from . import api as _api
from .api import bucket_ids_of, bucket_of, intersecting_buckets, partition_buckets
from .graph import SENTINEL, BucketMeta, GraphIndex, StoreView, create_index
from .params import CapacityError, DimensionMismatchError

__all__ = ["SENTINEL", "VectorStore", "BucketMeta", "GraphIndex", "StoreView", "append_batch", "bucket_ids_of",
           "bucket_of", "create_index", "intersecting_buckets", "new_adjacency", "partition_buckets"]


class VectorStore:
    """Append-only host store of fixed capacity (layout.py:22-79).

    Rows [0, count) are immutable once published; ``claim`` hands out unique
    contiguous ranges under a lock and ``count`` only advances when every row
    below it has been published, so a reader never sees a half-written row.
    """

    def __init__(self, capacity: int, dim: int):
        if capacity < 1 or dim < 1:
            raise ValueError("capacity and dim must be >= 1")
        self.X = np.zeros((capacity, dim), dtype="<f4")
        self.scalars = np.zeros(capacity, dtype="<f4")
        self.ids = np.full(capacity, -1, dtype="<i8")
        self._capacity = int(capacity)
        self._dim = int(dim)
        self._lock = threading.Lock()
        self._claimed = 0
        self._count = 0
        self._pending: dict[int, int] = {}  # published start -> end, not yet contiguous with count

    @property
    def capacity(self) -> int:
        return self._capacity

    @property
    def dim(self) -> int:
        return self._dim

    @property
    def count(self) -> int:
        return self._count

    def claim(self, n_rows: int) -> int:
        with self._lock:
            if self._claimed + n_rows > self._capacity:
                raise CapacityError(f"capacity exhausted: {self._claimed} claimed + {n_rows} requested > "
                                    f"{self._capacity}")
            start = self._claimed
            self._claimed += n_rows
            return start

    def publish(self, start: int, n_rows: int) -> None:
        with self._lock:
            self._pending[start] = start + n_rows
            while self._count in self._pending:
                self._count = self._pending.pop(self._count)


def new_adjacency(capacity: int, k_max: int) -> np.ndarray:
    """layout.py:177-178: an all-SENTINEL u32 [capacity x k_max] table."""
    return np.full((capacity, k_max), SENTINEL, dtype="<u4")


def append_batch(store, meta, vectors, scalars, ids=None) -> tuple[int, int]:
    """append_batch (layout.py:181-223): rows at the tail, [start, end) returned.

    ``store`` is a host ``VectorStore`` (written in place; ``meta``'s maps get
    the bucket ids, looked up on the device, before the count is published) or
    a device ``GraphIndex`` / its ``store`` view (appended on the device; the
    index owns its bucket maps, so ``meta`` is ignored there).
    """
    if isinstance(store, (GraphIndex, StoreView)):
        return _api.append_batch(store, vectors, scalars, ids=ids)
    V = np.asarray(vectors, dtype=np.float32)
    S = np.asarray(scalars, dtype=np.float32).reshape(-1)
    b = len(V)
    if b == 0:
        c = store.count
        return c, c
    if V.ndim != 2 or V.shape[1] != store.dim:
        raise DimensionMismatchError(f"vectors have shape {V.shape}, index dimension is {store.dim}")
    if len(S) != b:
        raise ValueError(f"{b} vectors but {len(S)} scalars")
    if not np.all(np.isfinite(S)):
        raise ValueError("scalars must be finite")
    start = store.claim(b)
    end = start + b
    store.X[start:end] = V
    store.scalars[start:end] = S
    store.ids[start:end] = np.arange(start, end) if ids is None else np.asarray(ids, dtype=np.int64)
    if meta is not None:
        bids = bucket_ids_of(meta, S)
        meta.index_to_bucket[start:end] = bids
        for off, bid in enumerate(bids.tolist()):
            meta.bucket_to_index[bid].append(start + off)
    store.publish(start, b)
    return start, end
