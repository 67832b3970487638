"""``bucketann.builder`` surface (reference builder.py:1-561).

``build_index`` is the one-call device build (api.py). The phase-level entry
points the reference exports run the same device phases on an explicit state:
the (store, meta) rows are imported into a scratch device index and
``grab_build_graph`` runs pass 1 (``build_local_phase``), pass 2
(``build_global_graph`` / ``exact_knn_graph``), ``grab_fuse`` the remote-edge
fusion and ``grab_reinforce`` the orphan repair -- the kernels of build.cu /
knn_tc.cu / descent.cu, not a host re-implementation.

``interleave_merge`` and ``topk_ids_by_distance`` are the reference's small
list / matrix utilities (the device does the same work inside k_local_merge
and the kNN rerank); they are exported for callers that use them directly.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .api import BuildReport, build_index
from .graph import SENTINEL, BucketMeta, GraphIndex, import_state
from .params import BuildParams

__all__ = ["BuildReport", "GlobalGraph", "LocalGraphDraft", "build_global_graph", "build_index", "build_local_phase",
           "exact_knn_graph", "fuse_remote_edges", "interleave_merge", "reinforce_reachability",
           "topk_ids_by_distance", "EXACT_GLOBAL_LIMIT"]

EXACT_GLOBAL_LIMIT = 100_000  # builder.py:33


@dataclass
class LocalGraphDraft:
    """Pass-1 output (builder.py:36-52), slot ids, SENTINEL-padded to k_max."""

    forward_rows: np.ndarray
    rows: np.ndarray
    necessary_counts: np.ndarray
    isolated: list = field(default_factory=list)


@dataclass
class GlobalGraph:
    """Distance-ranked rows over the whole store (builder.py:55-60)."""

    rows: np.ndarray
    k_g: int


def _rows_scalars(store):
    n = store.count
    return np.ascontiguousarray(store.X[:n], dtype="<f4"), np.ascontiguousarray(store.scalars[:n], dtype="<f4"), n


def _scratch_index(store, meta: BucketMeta | None, params: BuildParams, adjacency=None) -> GraphIndex:
    """Upload (store rows, bucket maps, adjacency) into a scratch device index.

    ``meta`` None: one bucket holding every row (the global pass ignores buckets)."""
    X, S, n = _rows_scalars(store)
    gi = GraphIndex(store.dim, max(n, 1), params)
    if meta is None:
        lo, hi = (float(S.min()), float(S.max())) if n else (0.0, 1.0)
        bounds = np.array([lo, hi if hi > lo else np.nextafter(np.float32(lo), np.float32(np.inf))], "<f4")
        i2b = np.zeros(n, np.int32)
        lists = [np.arange(n)]
    else:
        bounds = np.asarray(meta.boundaries, dtype="<f4")
        i2b = np.asarray(meta.index_to_bucket[:n], dtype=np.int32)
        lists = [np.asarray(b, dtype=np.int64) for b in meta.bucket_to_index]
    A = np.full((n, params.k_max), SENTINEL, "<u4") if adjacency is None else adjacency
    return import_state(gi, X, S, A, bounds, i2b, lists, n)


def _run_graph(gi: GraphIndex, k_g: int, refine_rounds: int, exact_limit: int, flags: int, dbg) -> L.BuildReportC:
    rep = L.BuildReportC()
    L.check(L.lib.grab_build_graph(gi.handle, int(k_g), int(refine_rounds), int(exact_limit), int(flags),
                                   C.byref(rep), C.byref(dbg) if dbg is not None else None))
    gi._touch()
    return rep


def build_local_phase(store, meta: BucketMeta, params: BuildParams, n_threads: int = 1) -> LocalGraphDraft:
    """Pass 1 (builder.py:237-261): exact in-bucket kNN per bucket, reverse lists,
    interleaved merge; singleton buckets are isolated. ``n_threads`` is accepted
    for signature parity (the GPU is the parallelism)."""
    del n_threads
    n = store.count
    K = params.k_max
    fwd = np.full((n, K), SENTINEL, "<u4")
    rows = np.full((n, K), SENTINEL, "<u4")
    nec = np.zeros(n, "<u4")
    if n:
        gi = _scratch_index(store, meta, params)
        dbg = L.BuildDebugC(L.ptr(fwd), L.ptr(rows), L.ptr(nec), None)
        _run_graph(gi, K, 0, EXACT_GLOBAL_LIMIT, L.GRAPH_LOCAL_ONLY, dbg)
    isolated = [int(b[0]) for b in meta.bucket_to_index if len(b) == 1]
    return LocalGraphDraft(forward_rows=fwd, rows=rows, necessary_counts=nec.astype(np.int32), isolated=isolated)


def build_global_graph(store, params: BuildParams, k_g: int | None = None, refine_rounds: int = 3,
                       exact_limit: int = EXACT_GLOBAL_LIMIT) -> GlobalGraph:
    """Pass 2 (builder.py:364-393): exact kNN when count <= exact_limit, else
    random init + ``refine_rounds`` NN-descent rounds; then the reverse merge."""
    kg = params.k_max if k_g is None else int(k_g)
    n = store.count
    G = np.full((n, kg), SENTINEL, "<u4")
    if n >= 2:
        gi = _scratch_index(store, None, params)
        dbg = L.BuildDebugC(None, None, None, L.ptr(G))
        _run_graph(gi, kg, refine_rounds, exact_limit, L.GRAPH_GLOBAL_ONLY, dbg)
    return GlobalGraph(rows=G, k_g=kg)


def exact_knn_graph(X, k: int) -> np.ndarray:
    """builder.py:116-127: exact kNN ids (no self loops), (dist, slot) order, on
    the device (pass 1 over one bucket holding every row)."""
    from .layout import VectorStore
    X = np.asarray(X, dtype=np.float32)
    n = len(X)
    kk = min(int(k), n - 1)
    if kk <= 0:
        return np.empty((n, 0), np.int64)
    st = VectorStore(n, X.shape[1])
    st.X[:] = X
    st.claim(n)
    st.publish(0, n)
    params = BuildParams(k_max=kk, k_local=kk)
    meta = BucketMeta(boundaries=np.array([0.0, 1.0], "<f4"), index_to_bucket=np.zeros(n, np.int32),
                      bucket_to_index=[list(range(n))])
    return build_local_phase(st, meta, params).forward_rows[:, :kk].astype(np.int64)


def fuse_remote_edges(draft: LocalGraphDraft, gg: GlobalGraph, store, meta: BucketMeta, params: BuildParams,
                      adjacency: np.ndarray) -> None:
    """builder.py:396-452 on the device: ``adjacency[:n] = draft.rows``, then the
    proximal / global remote edges from column ``necessary_counts[u]``; the
    result is written into ``adjacency`` in place like the reference."""
    n = store.count
    if n == 0:
        return
    gi = _scratch_index(store, meta, params, adjacency=np.ascontiguousarray(draft.rows[:n], dtype="<u4"))
    nec = np.ascontiguousarray(draft.necessary_counts[:n], dtype="<u4")
    G = np.ascontiguousarray(gg.rows[:n], dtype="<u4")
    L.check(L.lib.grab_fuse(gi.handle, L.ptr(nec), L.ptr(G), int(G.shape[1])))
    gi._touch()
    adjacency[:n] = gi._read(L.ARR_ADJ, 0, n, "<u4", (n, params.k_max))


def reinforce_reachability(index: GraphIndex) -> int:
    """builder.py:455-500 on the device index: give every zero-in-degree node an
    incoming edge (<= 4 rounds); returns the number of links added."""
    added = C.c_uint64(0)
    L.check(L.lib.grab_reinforce(index.handle, C.byref(added)))
    index._touch()
    return int(added.value)


def _random_init_graph(X, k: int, rng: np.random.Generator):
    """builder.py:330-335: ``rng.integers(0, n - 1, (n, k))`` shifted past the row
    itself, and the edges' squared distances. The draw consumes the caller's
    numpy Generator (its state advances exactly like the reference's); the
    distances are computed on the device (f64, returned as f32)."""
    X = np.asarray(X, dtype=np.float32)
    n = len(X)
    graph = rng.integers(0, n - 1, size=(n, k), dtype=np.int64)
    graph[graph >= np.arange(n)[:, None]] += 1  # avoid self
    from .api import sq_distances
    dists = np.stack([sq_distances(X[v], X[graph[v]]) for v in range(n)]).astype(np.float32) if n else \
        np.empty((0, k), np.float32)
    return graph, dists


def _reverse_merge_topk(graph, X, k_g: int, block: int = 4096) -> np.ndarray:
    """builder.py:338-361: union with the reverse edges, dedup, the k_g closest
    per node by (dist, slot) -- the device build's global-pass kernels over this
    graph (``grab_reverse_merge_raw``; ``block`` is the reference's host
    blocking and has no meaning here)."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    g = np.asarray(graph)
    n, k = g.shape
    g32 = np.where((g >= 0) & (g < n), g, SENTINEL).astype("<u4")
    out = np.empty((n, int(k_g)), "<u4")
    if n:
        L.check(L.lib.grab_reverse_merge_raw(0, L.ptr(X), n, X.shape[1], L.ptr(np.ascontiguousarray(g32)), k,
                                             int(k_g), L.ptr(out)))
    return out.astype(np.int64)


def interleave_merge(forward, reverse, k_max: int) -> list:
    """builder.py:130-153: forward[0], reverse[0], forward[1], ... without repeats."""
    out: list = []
    seen: set = set()
    for i in range(max(len(forward), len(reverse))):
        for src in (forward, reverse):
            if i < len(src) and src[i] not in seen:
                if len(out) == k_max:
                    return out
                seen.add(src[i])
                out.append(src[i])
    return out[:k_max]


def topk_ids_by_distance(dists, k: int) -> np.ndarray:
    """builder.py:90-113: per row, the k smallest columns ordered by (dist, col)."""
    d = np.asarray(dists)
    k = min(int(k), d.shape[1])
    cols = np.broadcast_to(np.arange(d.shape[1]), d.shape)
    return np.ascontiguousarray(np.lexsort((cols, d))[:, :k])
