"""Device-resident GraphIndex with reference-shaped host views.

The reference GraphIndex (layout.py:226-257) is a bag of numpy arrays. Here
the arrays live in B200 HBM in the bucket-slab layout owned by libgrab; the
attributes callers and tests read (``index.store.X``, ``index.adjacency``,
``index.meta.bucket_to_index`` ...) are materialised on demand in the
reference's slot order and cached until the next topology write.
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _lib as L
from .params import BuildParams

SENTINEL = np.uint32(0xFFFFFFFF)  # layout.py:19


@dataclass
class BucketMeta:
    """Boundaries + M_I2B + M_B2I (layout.py:82-104); plain host arrays."""

    boundaries: np.ndarray
    index_to_bucket: np.ndarray
    bucket_to_index: list

    @property
    def m(self) -> int:
        return len(self.boundaries) - 1

    @property
    def span(self) -> float:
        return float(self.boundaries[-1]) - float(self.boundaries[0])


class StoreView:
    """Read-only VectorStore facade (layout.py:22-79) over the device rows."""

    def __init__(self, index: "GraphIndex"):
        self._ix = index

    @property
    def capacity(self) -> int:
        return self._ix.capacity

    @property
    def dim(self) -> int:
        return self._ix.dim

    @property
    def count(self) -> int:
        return self._ix.count

    @property
    def X(self) -> np.ndarray:
        return self._ix._cached("X", self._ix._read_X)

    @property
    def scalars(self) -> np.ndarray:
        return self._ix._cached("S", self._ix._read_scalars)

    @property
    def ids(self) -> np.ndarray:
        return self._ix._ids


class GraphIndex:
    """Owning handle of one device index (one B200)."""

    def __init__(self, dim: int, capacity: int, params: BuildParams, device: int = 0, global_pass: str = "auto"):
        self.params = params
        self.device = device
        h = C.c_void_p()
        bp = to_c_params(params, global_pass)
        L.check(L.lib.grab_create(device, dim, capacity, C.byref(bp), C.byref(h)))
        self._h = h
        self._dim = dim
        self._capacity = capacity
        self._ids = np.full(capacity, -1, dtype="<i8")
        self._cache: dict = {}
        self._version = 0

    # -- lifecycle ---------------------------------------------------------
    def __del__(self):
        h = getattr(self, "_h", None)
        lib = getattr(L, "lib", None) if L is not None else None
        if h is not None and h.value and lib is not None:  # (module globals may be gone at interpreter exit)
            lib.grab_destroy(h)
            self._h = None

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def info(self) -> L.InfoC:
        inf = L.InfoC()
        L.check(L.lib.grab_get_info(self._h, C.byref(inf)))
        return inf

    def _touch(self) -> None:
        self._version += 1
        self._cache.clear()

    def _cached(self, key, fn):
        if key not in self._cache:
            self._cache[key] = fn()
        return self._cache[key]

    # -- shape -------------------------------------------------------------
    @property
    def count(self) -> int:
        return int(self.info().count)

    @property
    def dim(self) -> int:
        return self._dim

    @property
    def capacity(self) -> int:
        return self._capacity

    @property
    def built(self) -> bool:
        return bool(self.info().built)

    @property
    def store(self) -> StoreView:
        return StoreView(self)

    # -- materialised views (slot order, reference shapes) -------------------
    def _read(self, what: int, start: int, count: int, dtype, shape) -> np.ndarray:
        out = np.empty(shape, dtype=dtype)
        if count:
            L.check(L.lib.grab_read(self._h, what, start, count, L.ptr(out)))
        return out

    def _read_X(self) -> np.ndarray:
        n = self.count
        X = np.zeros((self._capacity, self._dim), dtype="<f4")
        X[:n] = self._read(L.ARR_X, 0, n, "<f4", (n, self._dim))
        X.setflags(write=False)
        return X

    def _read_scalars(self) -> np.ndarray:
        n = self.count
        s = np.zeros(self._capacity, dtype="<f4")
        s[:n] = self._read(L.ARR_SCALARS, 0, n, "<f4", (n,))
        s.setflags(write=False)
        return s

    def _read_adj(self) -> np.ndarray:
        n, k = self.count, self.params.k_max
        A = np.full((self._capacity, k), SENTINEL, dtype="<u4")
        A[:n] = self._read(L.ARR_ADJ, 0, n, "<u4", (n, k))
        A.setflags(write=False)
        return A

    def _read_meta(self):
        inf = self.info()
        if not inf.built:
            return None
        m = int(inf.m)
        b = self._read(L.ARR_BOUNDARIES, 0, m + 1, "<f4", (m + 1,))
        i2b = self._read(L.ARR_I2B, 0, self._capacity, "<i4", (self._capacity,))
        off = self._read(L.ARR_B2I_OFFSETS, 0, m + 1, "<u8", (m + 1,))
        flat = self._read(L.ARR_B2I_FLAT, 0, int(off[-1]), "<u4", (int(off[-1]),))
        lists = [flat[off[i]:off[i + 1]].astype(np.int64).tolist() for i in range(m)]
        return BucketMeta(boundaries=b, index_to_bucket=i2b, bucket_to_index=lists)

    @property
    def adjacency(self) -> np.ndarray:
        return self._cached("A", self._read_adj)

    @property
    def meta(self) -> BucketMeta | None:
        return self._cached("meta", self._read_meta)


GLOBAL_PASS = {"auto": 0, "exact": 1, "descent": 2}


def to_c_params(p: BuildParams, global_pass: str = "auto") -> L.BuildParamsC:
    """``global_pass`` (not a reference field): pass-2 candidate graph -- "auto" is the
    reference rule (exact kNN iff n <= 100 000, else NN-descent; builder.py:379-391)."""
    if global_pass not in GLOBAL_PASS:
        raise ValueError(f"unknown global_pass: {global_pass!r}")
    return L.BuildParamsC(k_max=p.k_max, k_local=p.k_local, bucket_capacity=p.bucket_capacity,
                          global_pass=GLOBAL_PASS[global_pass],
                          proximal_fraction=float(p.proximal_fraction), proximal_window=float(p.proximal_window),
                          alpha=float(p.alpha), rng_seed=int(p.rng_seed))


def create_index(dim: int, capacity: int, params: BuildParams, device: int = 0,
                 global_pass: str = "auto") -> GraphIndex:
    """create_index (layout.py:250-257): empty device index of fixed capacity."""
    return GraphIndex(dim, capacity, params, device, global_pass)


def import_state(index: GraphIndex, X, scalars, adjacency, boundaries, index_to_bucket, bucket_to_index,
                 count: int, ids=None) -> GraphIndex:
    """Upload a slot-space index state (reference GraphIndex arrays) into the device layout."""
    n = int(count)
    Xh = np.ascontiguousarray(np.asarray(X)[:n], dtype="<f4")
    Sh = np.ascontiguousarray(np.asarray(scalars)[:n], dtype="<f4")
    Ah = np.ascontiguousarray(np.asarray(adjacency)[:n], dtype="<u4")
    Bh = np.ascontiguousarray(boundaries, dtype="<f4")
    Ih = np.ascontiguousarray(np.asarray(index_to_bucket)[:n], dtype="<i4")
    m = len(Bh) - 1
    sizes = [len(x) for x in bucket_to_index]
    off = np.zeros(m + 1, dtype="<u8")
    off[1:] = np.cumsum(sizes)
    flat = np.ascontiguousarray(np.concatenate([np.asarray(x, dtype=np.int64) for x in bucket_to_index])
                                if n else np.zeros(0), dtype="<u4")
    L.check(L.lib.grab_import(index.handle, n, L.ptr(Xh), L.ptr(Sh), L.ptr(Ah), L.ptr(Bh), m, L.ptr(Ih),
                              L.ptr(flat), L.ptr(off)))
    index._ids[:n] = np.arange(n) if ids is None else np.asarray(ids)[:n]
    index._touch()
    return index


def from_reference(ref_index, device: int = 0) -> GraphIndex:
    """Upload a ``bucketann.GraphIndex`` (e.g. a reference-built graph) to the device layout."""
    p = ref_index.params
    params = BuildParams(k_max=p.k_max, k_local=p.k_local, bucket_capacity=p.bucket_capacity,
                         proximal_fraction=p.proximal_fraction, proximal_window=p.proximal_window,
                         alpha=p.alpha, rng_seed=p.rng_seed)
    st = ref_index.store
    g = GraphIndex(st.dim, st.capacity, params, device)
    if ref_index.meta is None:
        return g
    meta = ref_index.meta
    return import_state(g, st.X, st.scalars, ref_index.adjacency, meta.boundaries, meta.index_to_bucket,
                        meta.bucket_to_index, st.count, ids=st.ids)


# ---- GRAB v1 container (dataio.py:111-187) ----------------------------------
_HEADER = struct.Struct("<4sIQQIIIIB")


def save_index(index: GraphIndex, path) -> None:
    """Byte-identical to the reference's save_index for the same index state."""
    meta = index.meta
    if meta is None:
        raise ValueError("cannot save an index that has never been built")
    n = index.count
    st = index.store
    with open(path, "wb") as f:
        f.write(_HEADER.pack(b"GRAB", 1, n, index.capacity, index.dim, index.params.k_max, index.params.k_local,
                             meta.m, 0))
        f.write(st.X[:n].astype("<f4", copy=False).tobytes())
        f.write(st.scalars[:n].astype("<f4", copy=False).tobytes())
        f.write(index.adjacency[:n].astype("<u4", copy=False).tobytes())
        f.write(meta.boundaries.astype("<f4", copy=False).tobytes())
        f.write(meta.index_to_bucket[:n].astype("<u4", copy=False).tobytes())


def load_index(path, params: BuildParams | None = None, device: int = 0) -> GraphIndex:
    """Read a GRAB v1 container straight into device memory."""
    raw = Path(path).read_bytes() if not isinstance(path, (bytes, bytearray, memoryview)) else bytes(path)
    if raw[:4] != b"GRAB":
        raise ValueError(f"not an index container: {path if isinstance(path, (str, Path)) else '<bytes>'}")
    _, version, n, n_cap, d, k_max, k_local, m, metric = _HEADER.unpack_from(raw, 0)
    if version != 1:
        raise ValueError(f"unsupported container version {version}")
    if metric != 0:
        raise ValueError(f"unsupported metric code {metric}")
    off = _HEADER.size
    views = []
    for dt, cnt in (("<f4", n * d), ("<f4", n), ("<u4", n * k_max), ("<f4", m + 1), ("<u4", n)):
        a = np.frombuffer(raw, dtype=dt, count=cnt, offset=off)
        off += a.nbytes
        views.append(a)
    X, S, A, B, I = views
    params = params or BuildParams(k_max=k_max, k_local=k_local)
    g = GraphIndex(d, n_cap, params, device)
    i2b = I.astype("<i4")
    order = np.argsort(i2b, kind="stable")
    counts = np.bincount(i2b, minlength=m)
    lists, pos = [], 0
    for c in counts.tolist():
        lists.append(order[pos:pos + c])
        pos += c
    return import_state(g, X.reshape(n, d), S, A.reshape(n, k_max), B, i2b, lists, n)
