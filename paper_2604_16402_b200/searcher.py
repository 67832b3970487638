"""``bucketann.searcher`` surface (reference searcher.py:1-248).

``search`` / ``search_batch`` run the persistent warp-per-query kernel
(csrc/search.cu) through ``grab_search``. ``derive_query_seed`` is the
SeedSequence restatement the kernel itself uses (csrc/rng.cuh), called through
``grab_derive_seeds``. ``CandidateQueue`` is the reference's bounded
(dist, slot) queue as a host value type for callers that use it directly; the
kernel keeps its own queue in shared memory (search.cu ``admit``).
"""
from __future__ import annotations

import numpy as np

from . import _lib as L
from .api import BatchResult, SearchResult, SearchStats, search, search_arrays, search_batch

__all__ = ["BatchResult", "CandidateQueue", "SearchResult", "SearchStats", "derive_query_seed", "search",
           "search_arrays", "search_batch"]


def derive_query_seed(rng_seed: int, ordinal: int) -> int:
    """searcher.py:85-87: SeedSequence([rng_seed, ordinal]).generate_state(1, u64)[0]."""
    if not 0 <= int(ordinal) < 2 ** 32:
        return int(np.random.SeedSequence([int(rng_seed), int(ordinal)]).generate_state(1, np.uint64)[0])
    o = np.array([int(ordinal)], dtype=np.uint32)
    out = np.empty(1, dtype=np.uint64)
    L.check(L.lib.grab_derive_seeds(int(rng_seed) & 0xFFFFFFFFFFFFFFFF, L.ptr(o), 1, L.ptr(out)))
    return int(out[0])


class CandidateQueue:
    """Bounded queue ascending by (dist, slot) with expansion flags (searcher.py:52-82)."""

    def __init__(self, capacity: int):
        self.capacity = int(capacity)
        self.slots = np.empty(0, dtype=np.int64)
        self.dists = np.empty(0, dtype=np.float64)
        self.expanded = np.empty(0, dtype=bool)

    def __len__(self) -> int:
        return len(self.slots)

    def admit(self, slots, dists) -> None:
        slots = np.asarray(slots, dtype=np.int64)
        if len(slots) == 0:
            return
        allS = np.append(self.slots, slots)
        allD = np.append(self.dists, np.asarray(dists, dtype=np.float64))
        allE = np.append(self.expanded, np.zeros(len(slots), dtype=bool))
        keep = np.lexsort((allS, allD))[: self.capacity]
        self.slots, self.dists, self.expanded = allS[keep], allD[keep], allE[keep]

    def frontier(self, width: int) -> np.ndarray:
        """Positions of the first ``width`` unexpanded entries (empty = converged)."""
        return np.nonzero(~self.expanded)[0][:width]

    def top_k(self, k: int):
        return self.slots[:k].copy(), self.dists[:k].copy()
