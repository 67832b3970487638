"""B200-native GRAB-ANNS range-filtered graph index (drop-in for ``bucketann``).

Every operation runs in hand-written sm_100a CUDA (libgrab.so, C ABI in
include/grab.h); Python only marshals arguments. There is no CPU fallback:
importing without the built library raises ImportError.

The module layout mirrors the reference package (``core``, ``layout``,
``builder``, ``searcher``, ``updater``, ``evaluate``, ``dataio``), so
``compat/bucketann`` can alias ``import bucketann`` to this package.
"""
from .params import (BuildParams, CapacityError, DimensionMismatchError, RangePredicate, SearchParams,
                     VectorRecord)
from .graph import SENTINEL, BucketMeta, GraphIndex, StoreView, create_index, from_reference, load_index, save_index
from .api import (BatchResult, BuildDraft, BuildReport, InsertReport, build_index, insert_batch, select_neighbors,
                  try_rewire, SearchResult, SearchStats, brute_force_arrays, brute_force_search, bucket_ids_of,
                  bucket_of, intersecting_buckets, partition_buckets, search, search_arrays, search_batch,
                  sq_distance, sq_distances)
from .layout import VectorStore, append_batch, new_adjacency
from .builder import (GlobalGraph, LocalGraphDraft, build_global_graph, build_local_phase, exact_knn_graph,
                      fuse_remote_edges, reinforce_reachability)
from .searcher import CandidateQueue, derive_query_seed
from .datasets import gen_synthetic, recall_at_k
from .dataio import FvecsFormatError, read_fvecs, read_scalars, write_fvecs, write_scalars
from .evaluate import EvalReport, GroundTruthCache, SweepSpec, run_sweep, scc_count
from . import builder, core, dataio, evaluate, layout, searcher, updater  # noqa: F401  (reference submodules)

__version__ = "0.1.0"

__all__ = [
    # the reference's public surface (bucketann/__init__.py:48-91)
    "BuildParams", "BuildReport", "BucketMeta", "CapacityError", "DimensionMismatchError", "EvalReport",
    "GraphIndex", "GroundTruthCache", "InsertReport", "RangePredicate", "SENTINEL", "SearchParams", "SearchResult",
    "SweepSpec", "VectorRecord", "VectorStore", "append_batch", "brute_force_search", "bucket_of",
    "build_global_graph", "build_index", "build_local_phase", "create_index", "gen_synthetic", "insert_batch",
    "intersecting_buckets", "load_index", "partition_buckets", "read_fvecs", "read_scalars", "recall_at_k",
    "run_sweep", "save_index", "scc_count", "search", "search_batch", "select_neighbors", "sq_distance",
    "sq_distances", "try_rewire", "write_fvecs", "write_scalars",
    # additions: array-level batch calls, phase-level helpers, device views
    "BatchResult", "BuildDraft", "CandidateQueue", "FvecsFormatError", "GlobalGraph", "LocalGraphDraft",
    "SearchStats", "StoreView", "brute_force_arrays", "bucket_ids_of", "derive_query_seed", "exact_knn_graph",
    "from_reference", "fuse_remote_edges", "new_adjacency", "reinforce_reachability", "search_arrays",
]
