"""Measurement harness on the device (reference evaluate.py).

* ``scc_count``          evaluate.py:60-119 -- counted by libgrab on the GPU
                         (trim + forward-max coloring + backward closure,
                         csrc/scc.cu) instead of a sequential Tarjan
* ``GroundTruthCache``   evaluate.py:138-204 -- same SHA-256 key and GTC1 file
                         format; misses are filled by the GPU brute force
* ``SweepSpec`` / ``EvalReport`` / ``run_sweep``  evaluate.py:207-307 -- same
                         grid, CSV columns and per-query seeds
                         (derive_query_seed(rng_seed, i)); each grid cell runs
                         as ONE batched device search, so ``qps`` is the batch
                         throughput and the latency columns are batch time / nq
* ``generate_ranges`` / ``recall_at_k``  evaluate.py:47-57, 122-135
"""
from __future__ import annotations

import csv
import hashlib
import json
import struct
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _lib as L
from .api import brute_force_arrays, brute_force_search, search_arrays
from .datasets import generate_ranges, recall_at_k
from .params import SearchParams

__all__ = ["scc_count", "GroundTruthCache", "SweepSpec", "EvalReport", "run_sweep", "generate_ranges",
           "recall_at_k"]


def scc_count(adjacency_or_index, live_count: int | None = None) -> int:
    """Strongly connected components of the live graph (SENTINEL and targets >=
    live_count ignored). Accepts a GraphIndex (counted in place on its device)
    or a slot-space adjacency array (uploaded)."""
    out = np.zeros(1, dtype=np.uint64)
    if hasattr(adjacency_or_index, "handle"):
        live = L.LIVE_ALL if live_count is None else int(live_count)
        L.check(L.lib.grab_scc_count(adjacency_or_index.handle, live, L.ptr(out)))
    else:
        a = np.ascontiguousarray(adjacency_or_index, dtype="<u4")
        n = len(a) if live_count is None else int(live_count)
        L.check(L.lib.grab_scc_count_raw(L.ptr(a), len(a), a.shape[1], n, L.ptr(out)))
    return int(out[0])


class GroundTruthCache:
    """Disk + memory cache of exact filtered results (evaluate.py:138-204)."""

    MAGIC = b"GTC1"

    def __init__(self, directory=None):
        self.directory = Path(directory) if directory else None
        if self.directory:
            self.directory.mkdir(parents=True, exist_ok=True)
        self._memo: dict[str, list[np.ndarray]] = {}

    @staticmethod
    def _key(store, queries, k, ranges, live_count) -> str:
        n = store.count if live_count is None else live_count
        h = hashlib.sha256()
        h.update(np.ascontiguousarray(store.X[:n]).tobytes())
        h.update(np.ascontiguousarray(store.scalars[:n]).tobytes())
        h.update(np.asarray(queries, dtype=np.float32).tobytes())
        h.update(struct.pack("<q", k))
        for r in ranges:
            h.update(struct.pack("<dd", r.lower, r.upper))
        return h.hexdigest()

    def get(self, store, queries, k: int, ranges, live_count: int | None = None) -> list[np.ndarray]:
        """evaluate.py:159-182: ``store`` is ``index.store`` as in the reference (a
        GraphIndex is accepted too); misses run the device brute force on the
        store's index."""
        index = store._ix if hasattr(store, "_ix") else store
        store = index.store
        key = self._key(store, queries, k, ranges, live_count)
        if key in self._memo:
            return self._memo[key]
        path = self.directory / f"{key}.gt" if self.directory else None
        if path and path.exists():
            truth = self._read(path)
        else:
            lo = np.array([r.lower for r in ranges], dtype=np.float64)
            hi = np.array([r.upper for r in ranges], dtype=np.float64)
            s, _, c = brute_force_arrays(index, np.asarray(queries, dtype=np.float32), lo, hi, k, live_count)
            truth = [s[i, : c[i]].astype(np.int64) for i in range(len(c))]
            if path:
                self._write(path, truth, k)
        self._memo[key] = truth
        return truth

    def _write(self, path: Path, truth, k: int) -> None:
        with open(path, "wb") as f:
            f.write(self.MAGIC)
            f.write(struct.pack("<II", len(truth), k))
            for slots in truth:
                f.write(struct.pack("<I", len(slots)))
                f.write(np.asarray(slots, dtype="<u4").tobytes())

    def _read(self, path: Path) -> list[np.ndarray]:
        raw = path.read_bytes()
        if raw[:4] != self.MAGIC:
            raise ValueError(f"not a ground-truth cache file: {path}")
        nq, _k = struct.unpack_from("<II", raw, 4)
        off, out = 12, []
        for _ in range(nq):
            (m,) = struct.unpack_from("<I", raw, off)
            off += 4
            out.append(np.frombuffer(raw, dtype="<u4", count=m, offset=off).astype(np.int64))
            off += 4 * m
        return out


@dataclass
class SweepSpec:
    """Cartesian grid for the bench harness (evaluate.py:207-217)."""

    selectivities: list = field(default_factory=lambda: [0.01, 0.1, 0.2, 1.0])
    itopk_values: list = field(default_factory=lambda: [128])
    search_widths: list = field(default_factory=lambda: [4])
    max_iterations_values: list = field(default_factory=lambda: [50])
    k: int = 10
    query_count: int = 100
    rng_seed: int = 0


_CSV_COLUMNS = ["selectivity", "k", "itopk", "search_width", "max_iterations", "recall", "qps", "mean_latency_us",
                "p99_latency_us", "dist_evals_per_query", "scc"]


@dataclass
class EvalReport:
    rows: list = field(default_factory=list)

    def write_csv(self, path) -> None:
        with open(path, "w", newline="") as f:
            w = csv.DictWriter(f, fieldnames=_CSV_COLUMNS)
            w.writeheader()
            w.writerows(self.rows)

    def write_json(self, path) -> None:
        Path(path).write_text(json.dumps(self.rows, indent=2))


def run_sweep(index, queries, spec: SweepSpec, *, gt_cache: GroundTruthCache | None = None) -> EvalReport:
    """evaluate.py:249-307 with every grid cell as one batched device search."""
    queries = np.asarray(queries, dtype=np.float32)[: spec.query_count]
    cache = gt_cache or GroundTruthCache(None)
    n = index.count
    scalars = index.store.scalars[:n]
    scc = scc_count(index, n)
    report = EvalReport()
    for sel in spec.selectivities:
        ranges = generate_ranges(scalars, sel, len(queries), spec.rng_seed)
        truth = cache.get(index.store, queries, spec.k, ranges)
        lo = np.array([r.lower for r in ranges], dtype=np.float64)
        hi = np.array([r.upper for r in ranges], dtype=np.float64)
        for itopk in spec.itopk_values:
            for width in spec.search_widths:
                for max_iter in spec.max_iterations_values:
                    p = SearchParams(k=spec.k, itopk=itopk, search_width=width, max_iterations=max_iter)
                    t0 = time.perf_counter()
                    r = search_arrays(index, queries, lo, hi, p, seed_base=spec.rng_seed)
                    el = time.perf_counter() - t0
                    rec = [recall_at_k(r.slots[i, : r.counts[i]], truth[i], spec.k) for i in range(len(queries))]
                    per = el / max(len(queries), 1)
                    report.rows.append({
                        "selectivity": sel, "k": spec.k, "itopk": itopk, "search_width": width,
                        "max_iterations": max_iter, "recall": float(np.nanmean(rec)) if len(rec) else float("nan"),
                        "qps": len(queries) / el if el > 0 else 0.0, "mean_latency_us": per * 1e6,
                        "p99_latency_us": per * 1e6,
                        "dist_evals_per_query": float(np.mean(r.stats["dist_evals"])) if len(queries) else 0.0,
                        "scc": scc})
    return report
