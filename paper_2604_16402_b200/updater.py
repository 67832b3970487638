"""``bucketann.updater`` surface (reference updater.py:1-324): the append-only
batched insertion pipeline (csrc/insert.cu) and its pruning primitives."""
from __future__ import annotations

from .api import InsertReport, insert_batch, select_neighbors, try_rewire

__all__ = ["InsertReport", "insert_batch", "select_neighbors", "try_rewire", "CANDIDATE_LOCAL_FACTOR",
           "CANDIDATE_SEARCH_ITOPK", "CANDIDATE_SEARCH_WIDTH", "CANDIDATE_SEARCH_MAX_ITER"]

# updater.py:25-28 (the device pipeline uses the same constants, insert.cu)
CANDIDATE_LOCAL_FACTOR = 2
CANDIDATE_SEARCH_ITOPK = 128
CANDIDATE_SEARCH_WIDTH = 4
CANDIDATE_SEARCH_MAX_ITER = 50
