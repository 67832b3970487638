"""Operations of the drop-in surface, each one call into libgrab.

Reference functions replaced (paths under /root/reference/pkg/src/bucketann):
  search / search_batch          searcher.py:156-248
  brute_force_search             evaluate.py:22-44
  bucket_of / intersecting_buckets / bucket_ids_of   layout.py:157-174
  build_index                    builder.py:503-548
  insert_batch                   updater.py:154-263
  select_neighbors / try_rewire  updater.py:49-123

Inputs may be numpy arrays (host; copied by the library) or CUDA torch tensors
(device-resident; no host round trip).
"""
from __future__ import annotations

import ctypes as C
import time
from collections.abc import Sequence
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .graph import BucketMeta, GraphIndex, StoreView, create_index
from .params import BuildParams, DimensionMismatchError, RangePredicate, SearchParams


@dataclass(slots=True)
class SearchStats:
    """searcher.py:22-31 (+ ``expanded``: frontier nodes popped)."""

    iterations: int = 0
    dist_evals: int = 0
    seed_evals: int = 0
    gathered: int = 0
    in_range_new: int = 0
    precheck_rejected: int = 0
    seed_attempts: int = 0
    expanded: int = 0
    elapsed_s: float = 0.0


@dataclass(slots=True)
class SearchResult:
    """searcher.py:34-49: ascending (distance, slot); ``truncated`` when 0 < len < k."""

    slots: np.ndarray
    sq_dists: np.ndarray
    truncated: bool
    stats: SearchStats = field(default_factory=SearchStats)

    def __len__(self) -> int:
        return len(self.slots)


@dataclass
class BatchResult:
    """Array form of a query batch: slots/dists [nq, k] (-1 / NaN padded), counts, stats."""

    slots: np.ndarray
    dists: np.ndarray
    counts: np.ndarray
    stats: np.ndarray | None
    elapsed_s: float

    def to_results(self, k: int) -> "ResultList":
        return ResultList(self, k)


class _BatchItem(SearchResult):
    """A search_batch result: slots / sq_dists are views of the batch rows and
    ``stats`` (a SearchStats) is built on first access from the batch's counters,
    so iterating a 10K-query batch creates one small object per query."""

    __slots__ = ("_src", "_i")

    @property
    def stats(self) -> SearchStats:
        return self._src._stats_of(self._i)


_new_item = object.__new__


class ResultList(Sequence):
    """search_batch's list of SearchResult (searcher.py:236-248), materialised per
    item on access: the batch arrays stay as they came back from the kernel and
    each SearchResult's slots / sq_dists are views of its row, so returning a
    10K-query batch costs nothing per query until a caller reads it."""

    def __init__(self, batch: BatchResult, k: int):
        self._b = batch
        self._k = k
        self._counts = np.asarray(batch.counts).tolist()
        self._per = batch.elapsed_s / max(len(self._counts), 1)
        self._stats_rows = None
        self._full = None  # per-row views of slots / dists (rows with count == k)

    def __len__(self) -> int:
        return len(self._counts)

    def _stats_of(self, i: int) -> SearchStats:
        if self._b.stats is None:
            return SearchStats(elapsed_s=self._per)
        if self._stats_rows is None:
            self._stats_rows = np.asarray(self._b.stats).tolist()
        return SearchStats(*self._stats_rows[i], elapsed_s=self._per)

    def _item(self, i: int) -> SearchResult:
        if self._full is None:
            self._full = (list(self._b.slots), list(self._b.dists))
        c = self._counts[i]
        r = _new_item(_BatchItem)
        if c == self._k:
            r.slots = self._full[0][i]
            r.sq_dists = self._full[1][i]
            r.truncated = False
        else:
            r.slots = self._b.slots[i, :c]
            r.sq_dists = self._b.dists[i, :c]
            r.truncated = 0 < c
        r._src = self
        r._i = i
        return r

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self._item(j) for j in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        return self._item(i)

    def __iter__(self):
        for i in range(len(self)):
            yield self._item(i)


def _is_dev(a) -> bool:
    return hasattr(a, "is_cuda") and bool(a.is_cuda)


def _check_dev(t, name: str, dtype: str, ndim: int, index: GraphIndex):
    """Device-path argument checks (the host path gets the same from numpy
    conversion): libgrab reads raw pointers, so dtype / rank / device must match."""
    import torch
    want = getattr(torch, dtype)
    if not (hasattr(t, "is_cuda") and t.is_cuda):
        raise ValueError(f"{name} must be a CUDA tensor when the other inputs are")
    if t.dtype != want:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if t.dim() != ndim:
        raise DimensionMismatchError(f"{name} must be {ndim}-D, got shape {tuple(t.shape)}")
    if t.device.index != index.device:
        raise ValueError(f"{name} is on cuda:{t.device.index}, the index on cuda:{index.device}")
    return t.contiguous()


def _is_pinned(a) -> bool:
    return hasattr(a, "is_pinned") and not _is_dev(a) and bool(a.is_pinned())


def _pinned_empty(shape, dtype) -> np.ndarray:
    """numpy view of a page-locked host buffer (torch's pinned caching allocator)."""
    import torch
    dt = np.dtype(dtype)
    n = int(np.prod(shape))
    buf = torch.empty(max(n * dt.itemsize, 1), dtype=torch.uint8, pin_memory=True)
    return buf.numpy()[: n * dt.itemsize].view(dt).reshape(shape)


def _live(live_count) -> int:
    return L.LIVE_ALL if live_count is None else int(live_count)


def _search_params_c(params: SearchParams) -> L.SearchParamsC:
    return L.SearchParamsC(k=params.k, itopk=params.itopk, search_width=params.search_width,
                           max_iterations=params.max_iterations, seed_count=params.seed_count or 0)


def search_arrays(index: GraphIndex, queries, lower, upper, params: SearchParams, *, seeds=None,
                  seed_base: int | None = None, ordinal0: int = 0, live_count=None, stats: bool = True,
                  stream=None) -> BatchResult:
    """Batched filtered search with per-query ranges.

    ``lower``/``upper``: per-query bounds (arrays of length nq) or scalars (one
    shared range). Per-query RNG seed = ``seeds[i]`` if given, else
    derive_query_seed(seed_base, ordinal0 + i) (searcher.py:85-87; seed_base
    defaults to params.rng_seed, i.e. search_batch semantics).
    """
    dev = _is_dev(queries)
    if dev:
        import torch
        Q = _check_dev(queries, "queries", "float32", 2, index)
        nq, d = Q.shape
        lo = torch.as_tensor(lower, dtype=torch.float64, device=Q.device).reshape(-1).contiguous()
        hi = torch.as_tensor(upper, dtype=torch.float64, device=Q.device).reshape(-1).contiguous()
        sd = None if seeds is None else torch.as_tensor(seeds, dtype=torch.uint64, device=Q.device).contiguous()
        k = params.k
        slots = torch.empty((nq, k), dtype=torch.int64, device=Q.device)
        dists = torch.empty((nq, k), dtype=torch.float64, device=Q.device)
        counts = torch.empty(nq, dtype=torch.int32, device=Q.device)
        st = torch.empty((nq, len(L.STAT_FIELDS)), dtype=torch.int32, device=Q.device) if stats else None
        mem = L.MEM_DEVICE
        s_ptr = stream if stream is not None else torch.cuda.current_stream(Q.device).cuda_stream
    else:
        Q = np.ascontiguousarray(queries, dtype=np.float32)
        if Q.ndim == 1:
            Q = Q.reshape(1, -1)
        nq, d = Q.shape
        lo = np.ascontiguousarray(np.atleast_1d(np.asarray(lower, dtype=np.float64)))
        hi = np.ascontiguousarray(np.atleast_1d(np.asarray(upper, dtype=np.float64)))
        sd = None if seeds is None else np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
        k = params.k
        # page-locked queries (a pinned torch CPU tensor) get page-locked result
        # buffers too, so both copies are plain DMA (no pageable staging)
        alloc = _pinned_empty if _is_pinned(queries) else np.empty
        slots = alloc((nq, k), np.int64)
        dists = alloc((nq, k), np.float64)
        counts = alloc(nq, np.uint32)
        st = alloc(nq, L.STATS_DTYPE) if stats else None
        mem = L.MEM_HOST
        s_ptr = None
    if d != index.dim:
        raise DimensionMismatchError(f"query dimension {d} vs index dimension {index.dim}")
    stride = 0 if len(lo) == 1 else 1
    if len(lo) not in (1, nq) or len(hi) != len(lo):
        raise ValueError("lower/upper must be scalars or have one entry per query")
    base = params.rng_seed if seed_base is None else seed_base
    t0 = time.perf_counter()
    if nq:
        L.check(L.lib.grab_search(index.handle, L.ptr(Q), nq, L.ptr(lo), L.ptr(hi), stride,
                                  C.byref(_search_params_c(params)), L.ptr(sd), int(base), int(ordinal0),
                                  _live(live_count), L.ptr(slots), L.ptr(dists), L.ptr(counts), L.ptr(st), mem,
                                  s_ptr))
    el = time.perf_counter() - t0
    return BatchResult(slots, dists, counts, st, el)


def search(index: GraphIndex, query, params: SearchParams, *, live_count=None) -> SearchResult:
    """searcher.py:156-233: one query, RNG seeded with params.rng_seed directly."""
    q = np.asarray(query, dtype=np.float32).reshape(1, -1)
    r = search_arrays(index, q, params.range.lower, params.range.upper, params,
                      seeds=np.array([params.rng_seed], dtype=np.uint64), live_count=live_count)
    res = r.to_results(params.k)[0]
    return SearchResult(res.slots.copy(), res.sq_dists.copy(), res.truncated, res.stats)


def search_batch(index: GraphIndex, queries, params: SearchParams, *, live_count=None) -> Sequence:
    """searcher.py:236-248: shared range, seeds derive_query_seed(params.rng_seed, i).

    Returns a sequence of SearchResult (``ResultList``, built per item on access).
    A page-locked torch CPU tensor of queries takes the zero-copy path."""
    Q = queries if _is_pinned(queries) else np.asarray(queries, dtype=np.float32)
    if len(Q) == 0:
        return []
    r = search_arrays(index, Q, params.range.lower, params.range.upper, params, live_count=live_count)
    return r.to_results(params.k)


def brute_force_arrays(index: GraphIndex, queries, lower, upper, k: int, live_count=None):
    """Exact range-filtered top-k for a batch: (slots [nq,k] -1 padded, dists, counts)."""
    Q = np.ascontiguousarray(queries, dtype=np.float32)
    if Q.ndim == 1:
        Q = Q.reshape(1, -1)
    nq, d = Q.shape
    if d != index.dim:
        raise DimensionMismatchError(f"query dimension {d} vs index dimension {index.dim}")
    lo = np.ascontiguousarray(np.atleast_1d(np.asarray(lower, dtype=np.float64)))
    hi = np.ascontiguousarray(np.atleast_1d(np.asarray(upper, dtype=np.float64)))
    stride = 0 if len(lo) == 1 else 1
    slots = np.empty((nq, k), dtype=np.int64)
    dists = np.empty((nq, k), dtype=np.float64)
    counts = np.empty(nq, dtype=np.uint32)
    if nq:
        L.check(L.lib.grab_brute_force(index.handle, L.ptr(Q), nq, L.ptr(lo), L.ptr(hi), stride, k,
                                       _live(live_count), L.ptr(slots), L.ptr(dists), L.ptr(counts), L.MEM_HOST,
                                       None))
    return slots, dists, counts


def brute_force_search(store, query, k: int, rng: RangePredicate, live_count=None):
    """evaluate.py:22-44 over the index's rows (``store`` = index.store or the index)."""
    index = store._ix if hasattr(store, "_ix") else store
    s, d, c = brute_force_arrays(index, np.asarray(query, dtype=np.float32).reshape(1, -1), rng.lower, rng.upper,
                                 k, live_count)
    n = int(c[0])
    return s[0, :n].copy(), d[0, :n].copy()


def sq_distances(q, rows) -> np.ndarray:
    """core.py:25-38 on the device: f64-accumulated squared L2 of q to each row.

    Uses the same lane split and reduction tree as the search and brute-force
    kernels, so a distance returned by search equals sq_distance() bit for bit.
    """
    q = np.asarray(q)
    rows = np.asarray(rows)
    if rows.ndim != 2 or q.ndim != 1 or rows.shape[1] != q.shape[0]:
        raise DimensionMismatchError(f"shape mismatch: query {q.shape} vs rows {rows.shape}")
    qf = np.ascontiguousarray(q, dtype=np.float32)
    rf = np.ascontiguousarray(rows, dtype=np.float32)
    out = np.empty(len(rf), dtype=np.float64)
    if len(rf):
        L.check(L.lib.grab_sq_distances(L.ptr(qf), L.ptr(rf), len(rf), rf.shape[1], L.ptr(out)))
    return out


def sq_distance(a, b) -> float:
    """core.py:41-47."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape or a.ndim != 1:
        raise DimensionMismatchError(f"shape mismatch: {a.shape} vs {b.shape}")
    return float(sq_distances(a, b.reshape(1, -1))[0])


# ---- bucket selection (layout.py:157-174) -----------------------------------
def bucket_ids_of(meta, scalars) -> np.ndarray:
    index = meta if isinstance(meta, GraphIndex) else None
    s = np.ascontiguousarray(np.atleast_1d(np.asarray(scalars, dtype=np.float32)))
    out = np.empty(len(s), dtype=np.int32)
    if len(s) == 0:
        return out
    if index is not None:
        L.check(L.lib.grab_bucket_ids(index.handle, L.ptr(s), len(s), L.ptr(out), L.MEM_HOST, None))
        return out
    b = np.ascontiguousarray(meta.boundaries, dtype=np.float32)
    L.check(L.lib.grab_bucket_ids_raw(L.ptr(b), len(b) - 1, L.ptr(s), len(s), L.ptr(out)))
    return out


def partition_buckets(scalars, target_capacity: int, *, strategy: str = "quantile", capacity: int | None = None,
                      device: int = 0) -> BucketMeta:
    """partition_buckets (layout.py:107-154) on the device: quantile (sorted
    cuts, np.round half-even) or width (f32 linspace) edges, np.unique-collapsed;
    index_to_bucket sized to ``capacity`` (-1 past n); members in slot order."""
    if strategy not in _STRATEGY:
        raise ValueError(f"unknown bucket strategy: {strategy!r}")
    s = np.ascontiguousarray(np.asarray(scalars, dtype=np.float32).reshape(-1))
    n = len(s)
    if n < 1:
        raise ValueError("cannot partition an empty scalar set")
    if target_capacity < 1:
        raise ValueError("target_capacity must be >= 1")
    cap_b = -(-n // int(target_capacity)) + 1
    edges = np.empty(max(cap_b, 2), dtype="<f4")
    m = C.c_uint32(0)
    ids = np.empty(n, dtype="<i4")
    L.check(L.lib.grab_partition(int(device), L.ptr(s), n, int(target_capacity), _STRATEGY[strategy], L.ptr(edges),
                                 len(edges), C.byref(m), L.ptr(ids), L.MEM_HOST, None))
    mm = int(m.value)
    cap = n if capacity is None else int(capacity)
    i2b = np.full(cap, -1, dtype="<i4")
    i2b[:n] = ids
    order = np.argsort(ids, kind="stable")
    cuts = np.searchsorted(ids[order], np.arange(mm + 1))
    lists = [order[cuts[b]:cuts[b + 1]].tolist() for b in range(mm)]
    return BucketMeta(boundaries=edges[: mm + 1].copy(), index_to_bucket=i2b, bucket_to_index=lists)


def bucket_of(meta, s: float) -> int:
    return int(bucket_ids_of(meta, np.array([s], dtype=np.float32))[0])


def intersecting_buckets(meta, rng: RangePredicate) -> tuple[int, int]:
    lo = np.array([rng.lower], dtype=np.float64)
    hi = np.array([rng.upper], dtype=np.float64)
    a = np.empty(1, dtype=np.int32)
    b = np.empty(1, dtype=np.int32)
    if isinstance(meta, GraphIndex):
        L.check(L.lib.grab_bucket_select(meta.handle, L.ptr(lo), L.ptr(hi), 1, L.ptr(a), L.ptr(b), L.MEM_HOST, None))
    else:
        bd = np.ascontiguousarray(meta.boundaries, dtype=np.float32)
        L.check(L.lib.grab_bucket_select_raw(L.ptr(bd), len(bd) - 1, L.ptr(lo), L.ptr(hi), 1, L.ptr(a), L.ptr(b)))
    return int(a[0]), int(b[0])


# ---- build_index (builder.py:503-548) -----------------------------------------
@dataclass
class BuildReport:
    """builder.py:63-76."""

    n: int = 0
    m: int = 0
    phase1_seconds: float = 0.0
    phase2_seconds: float = 0.0
    fuse_seconds: float = 0.0
    total_seconds: float = 0.0
    bucket_sizes: list = field(default_factory=list)
    isolated_nodes: int = 0
    cross_bucket_edge_ratio: float = 0.0
    global_pass: str = "exact"  # (ours) what pass 2 ran: "exact" kNN or "descent"

    def to_dict(self) -> dict:
        return dict(self.__dict__)


@dataclass
class BuildDraft:
    """Intermediate graphs of a build (LocalGraphDraft + GlobalGraph rows, slot ids)."""

    forward_rows: np.ndarray
    rows: np.ndarray
    necessary_counts: np.ndarray
    global_rows: np.ndarray


_STRATEGY = {"quantile": 0, "width": 1}


def build_index(vectors, scalars, params: BuildParams, *, capacity: int | None = None, headroom: float = 2.0,
                bucket_strategy: str = "quantile", n_threads: int = 1, k_g: int | None = None,
                refine_rounds: int = 3, device: int = 0, return_draft: bool = False, global_pass: str = "auto"):
    """Full static build on the device: partition, slab layout, pass 1, pass 2, fuse, repair.

    ``global_pass`` (ours): "auto" follows the reference (exact global kNN for
    n <= 100 000, random init + ``refine_rounds`` NN-descent rounds above);
    "exact" / "descent" force one.

    Returns (GraphIndex, BuildReport) like the reference, plus a BuildDraft when
    ``return_draft``. ``n_threads`` is accepted for signature parity (the GPU is
    the parallelism).
    """
    del n_threads
    if bucket_strategy not in _STRATEGY:
        raise ValueError(f"unknown bucket strategy: {bucket_strategy!r}")
    dev = _is_dev(vectors)
    if dev:
        import torch
        V = vectors.contiguous()
        S = scalars.contiguous()
        if V.dtype != torch.float32 or V.dim() != 2:
            raise DimensionMismatchError(f"vectors must be a 2-D float32 tensor, got {V.dtype} {tuple(V.shape)}")
        if S.dtype != torch.float32 or S.dim() != 1 or S.device != V.device:
            raise ValueError("scalars must be a 1-D float32 tensor on the vectors' device")
        n, dim = V.shape
        if len(S) != n:
            raise ValueError(f"{n} vectors but {len(S)} scalars")
        if not bool(torch.isfinite(S).all()):
            raise ValueError("scalars must be finite")
        torch.cuda.current_stream(V.device).synchronize()  # the library works on its own stream
        mem = L.MEM_DEVICE
    else:
        V = np.ascontiguousarray(vectors, dtype=np.float32)
        S = np.ascontiguousarray(scalars, dtype=np.float32)
        if V.ndim != 2:
            raise DimensionMismatchError(f"vectors must be 2-D, got {V.shape}")
        n, dim = V.shape
        if len(S) != n:
            raise ValueError(f"{n} vectors but {len(S)} scalars")
        if not np.all(np.isfinite(S)):
            raise ValueError("scalars must be finite")
        mem = L.MEM_HOST
    if capacity is None:
        capacity = max(int(n * headroom), n)
    index = create_index(dim, capacity, params, device, global_pass)
    kg = params.k_max if k_g is None else int(k_g)
    rep = L.BuildReportC()
    dbg = None
    draft = None
    if return_draft:
        draft = BuildDraft(np.empty((n, params.k_max), "<u4"), np.empty((n, params.k_max), "<u4"),
                           np.empty(n, "<u4"), np.empty((n, kg), "<u4"))
        dbg = L.BuildDebugC(L.ptr(draft.forward_rows), L.ptr(draft.rows), L.ptr(draft.necessary_counts),
                            L.ptr(draft.global_rows))
    L.check(L.lib.grab_build_ex(index.handle, L.ptr(V), L.ptr(S), n, _STRATEGY[bucket_strategy], kg,
                                refine_rounds, mem, C.byref(rep), C.byref(dbg) if dbg is not None else None))
    index._ids[:n] = np.arange(n)
    index._touch()
    m = int(rep.m)
    # bucket sizes from the M_B2I offsets alone (the full meta view is built lazily)
    off = index._read(L.ARR_B2I_OFFSETS, 0, m + 1, "<u8", (m + 1,)) if m else np.zeros(1, "<u8")
    report = BuildReport(n=int(rep.n), m=m, phase1_seconds=rep.phase1_seconds,
                         phase2_seconds=rep.phase2_seconds, fuse_seconds=rep.fuse_seconds,
                         total_seconds=rep.total_seconds,
                         bucket_sizes=np.diff(off.astype(np.int64)).tolist(),
                         isolated_nodes=int(rep.isolated_nodes),
                         cross_bucket_edge_ratio=float(rep.cross_bucket_edge_ratio),
                         global_pass="descent" if rep.global_descent else "exact")
    if return_draft:
        return index, report, draft
    return index, report


# ---- insert_batch (updater.py:154-263) ----------------------------------------
@dataclass
class InsertReport:
    """updater.py:31-46."""

    batch_size: int = 0
    bulk_built: int = 0
    forward_accepted: int = 0
    forward_rejected: int = 0
    reverse_accepted: int = 0
    reverse_rejected: int = 0
    evictions_necessary: int = 0
    evictions_redundant: int = 0
    forced_links: int = 0
    rewired_rows: Sequence = field(default_factory=list)
    wall_time_s: float = 0.0
    phase_seconds: dict = field(default_factory=dict)

    def to_dict(self) -> dict:
        d = dict(self.__dict__)
        if isinstance(d["rewired_rows"], RowList):
            d["rewired_rows"] = d["rewired_rows"].tolist()
        return d


class RowList(Sequence):
    """InsertReport.rewired_rows (updater.py:42,261: a sorted list of slots),
    backed by the library's uint32 array: building a Python list of ~1M ints
    cost more than the device work of a 100K batch. Compares equal to a list
    with the same items; ``tolist()`` / ``np.asarray`` give the plain forms."""

    __slots__ = ("_a",)

    def __init__(self, a: np.ndarray):
        self._a = a

    def __len__(self) -> int:
        return len(self._a)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return self._a[i].astype(np.int64).tolist()
        return int(self._a[i])

    def __iter__(self):
        return iter(self._a.astype(np.int64).tolist())

    def __contains__(self, v) -> bool:
        i = int(np.searchsorted(self._a, v))
        return i < len(self._a) and int(self._a[i]) == v

    def __eq__(self, other) -> bool:
        if isinstance(other, RowList):
            return np.array_equal(self._a, other._a)
        if isinstance(other, (list, tuple, np.ndarray)):
            return len(other) == len(self._a) and np.array_equal(self._a, np.asarray(other))
        return NotImplemented

    def __array__(self, dtype=None, copy=None):
        return self._a.astype(dtype or np.int64)

    def tolist(self) -> list:
        return self._a.astype(np.int64).tolist()

    def __repr__(self) -> str:
        return f"RowList({self._a.tolist()!r})" if len(self._a) <= 20 else f"RowList(<{len(self._a)} rows>)"


_INSERT_PHASES = ["append", "bucket_candidates", "candidate_search", "forward_select", "reverse_rewire", "heal"]


def insert_batch(index: GraphIndex, vectors, scalars, *, ids=None, search_itopk: int = 128) -> InsertReport:
    """Integrate one batch on the device: append, candidates, forward pruning, reverse rewiring, healing."""
    dev = _is_dev(vectors)
    if dev:
        import torch
        V = _check_dev(vectors, "vectors", "float32", 2, index)
        S = _check_dev(scalars, "scalars", "float32", 1, index)
        if not bool(torch.isfinite(S).all()):
            raise ValueError("scalars must be finite")
        torch.cuda.current_stream(V.device).synchronize()  # the library works on its own stream
        b = V.shape[0]
        mem = L.MEM_DEVICE
        Ih = None if ids is None else np.ascontiguousarray(ids.cpu().numpy() if hasattr(ids, "cpu") else ids,
                                                           dtype=np.int64)
    else:
        V = np.asarray(vectors, dtype=np.float32)
        S = np.ascontiguousarray(np.asarray(scalars, dtype=np.float32).reshape(-1))
        b = len(V)
        mem = L.MEM_HOST
        Ih = None if ids is None else np.ascontiguousarray(ids, dtype=np.int64)
    if b == 0:
        return InsertReport(batch_size=0)
    if V.ndim != 2 or V.shape[1] != index.dim:
        raise DimensionMismatchError(f"vectors have shape {tuple(V.shape)}, index dimension is {index.dim}")
    if len(S) != b:
        raise ValueError(f"{b} vectors but {len(S)} scalars")
    if not dev:
        V = np.ascontiguousarray(V)
        if not np.all(np.isfinite(S)):
            raise ValueError("scalars must be finite")
    rep = L.InsertReportC()
    L.check(L.lib.grab_insert(index.handle, L.ptr(V), L.ptr(S), L.ptr(Ih), b, int(search_itopk), mem,
                              C.byref(rep)))
    index._touch()
    n0 = index.count - b
    head = int(rep.bulk_built)  # an empty index bulk-builds its head with ids arange(head), like the reference
    index._ids[n0:n0 + b] = np.arange(n0, n0 + b)
    if Ih is not None:
        index._ids[n0 + head:n0 + b] = Ih[head:]
    rw = np.empty(int(rep.n_rewired), dtype=np.uint32)
    nout = C.c_uint64()
    if len(rw):
        L.check(L.lib.grab_last_rewired(index.handle, L.ptr(rw), len(rw), C.byref(nout)))
    return InsertReport(batch_size=int(rep.batch_size), bulk_built=int(rep.bulk_built),
                        forward_accepted=int(rep.forward_accepted), forward_rejected=int(rep.forward_rejected),
                        reverse_accepted=int(rep.reverse_accepted), reverse_rejected=int(rep.reverse_rejected),
                        evictions_necessary=int(rep.evictions_necessary),
                        evictions_redundant=int(rep.evictions_redundant), forced_links=int(rep.forced_links),
                        rewired_rows=RowList(rw), wall_time_s=float(rep.wall_time_s),
                        phase_seconds={k: float(rep.phase_seconds[i]) for i, k in enumerate(_INSERT_PHASES)})


def append_batch(index: GraphIndex, vectors, scalars, ids=None) -> tuple[int, int]:
    """append_batch (layout.py:181-223) on the device index: rows, scalars, ids and
    bucket maps at the tail, adjacency of the new slots left SENTINEL (no edges);
    returns [start, end). The reference takes (store, meta, ...); here the index
    owns both. Needs a built index (bucket metadata)."""
    if isinstance(index, StoreView):
        index = index._ix
    V = np.asarray(vectors, dtype=np.float32)
    S = np.ascontiguousarray(np.asarray(scalars, dtype=np.float32).reshape(-1))
    b = len(V)
    if b == 0:
        c = index.count
        return c, c
    if V.ndim != 2 or V.shape[1] != index.dim:
        raise DimensionMismatchError(f"vectors have shape {tuple(V.shape)}, index dimension is {index.dim}")
    if len(S) != b:
        raise ValueError(f"{b} vectors but {len(S)} scalars")
    if not np.all(np.isfinite(S)):
        raise ValueError("scalars must be finite")
    V = np.ascontiguousarray(V)
    Ih = None if ids is None else np.ascontiguousarray(ids, dtype=np.int64)
    st, en = C.c_uint64(0), C.c_uint64(0)
    L.check(L.lib.grab_append(index.handle, L.ptr(V), L.ptr(S), L.ptr(Ih), b, L.MEM_HOST, C.byref(st), C.byref(en)))
    start, end = int(st.value), int(en.value)
    index._ids[start:end] = np.arange(start, end) if Ih is None else Ih
    index._touch()
    return start, end


def _rows_of(store) -> np.ndarray:
    X = store.X if hasattr(store, "X") else store
    return np.ascontiguousarray(X, dtype=np.float32)


def select_neighbors(store, target: int, candidates, row_capacity: int, alpha: float, fresh) -> list[int]:
    """updater.py:49-84 on the device (Eq.1 with the Eq.2 alpha^2 bias on fresh candidates)."""
    if not candidates:
        return []
    X = _rows_of(store)
    cs = np.ascontiguousarray([int(c[0]) for c in candidates], dtype=np.int64)
    cd = np.ascontiguousarray([float(c[1]) for c in candidates], dtype=np.float64)
    fr = np.ascontiguousarray([1 if int(c[0]) in fresh else 0 for c in candidates], dtype=np.uint8)
    out = np.empty(max(int(row_capacity), 1), dtype=np.int64)
    n = C.c_uint32()
    L.check(L.lib.grab_select_neighbors(L.ptr(X), X.shape[0], X.shape[1], int(target), L.ptr(cs), L.ptr(cd),
                                        L.ptr(fr), len(cs), int(row_capacity), float(alpha), L.ptr(out),
                                        C.byref(n)))
    return [int(x) for x in out[: n.value]]


def try_rewire(store, adjacency: np.ndarray, v: int, q: int, sq_dvq: float, alpha: float,
               k_local: int) -> tuple[bool, int]:
    """updater.py:87-123 on the device; mutates ``adjacency[v]`` in place like the reference."""
    X = _rows_of(store)
    row = np.ascontiguousarray(adjacency[v], dtype=np.uint32)
    acc = C.c_int32()
    pos = C.c_int32()
    L.check(L.lib.grab_try_rewire(L.ptr(X), X.shape[0], X.shape[1], L.ptr(row), len(row), int(v), int(q),
                                  float(sq_dvq), float(alpha), int(k_local), C.byref(acc), C.byref(pos)))
    adjacency[v] = row
    return bool(acc.value), int(pos.value)
