"""B200-native GRAB-ANNS range-filtered graph index (drop-in for ``bucketann``).

Every operation runs in hand-written sm_100a CUDA (libgrab.so, C ABI in
include/grab.h); Python only marshals arguments. There is no CPU fallback:
importing without the built library raises ImportError.
"""
from .params import (BuildParams, CapacityError, DimensionMismatchError, RangePredicate, SearchParams,
                     VectorRecord)
from .graph import SENTINEL, BucketMeta, GraphIndex, create_index, from_reference, load_index, save_index
from .graph import StoreView as VectorStore  # the device-resident store's reference-shaped view
from .api import (BatchResult, BuildDraft, BuildReport, InsertReport, append_batch, build_index, insert_batch,
                  select_neighbors,
                  try_rewire, SearchResult, SearchStats, brute_force_arrays, brute_force_search, bucket_ids_of,
                  bucket_of, intersecting_buckets, partition_buckets, search, search_arrays, search_batch,
                  sq_distance, sq_distances)
from .datasets import gen_synthetic, recall_at_k
from .dataio import FvecsFormatError, read_fvecs, read_scalars, write_fvecs, write_scalars
from .evaluate import EvalReport, GroundTruthCache, SweepSpec, run_sweep, scc_count

__version__ = "0.1.0"

__all__ = [
    "BatchResult", "BuildDraft", "BuildReport", "InsertReport", "build_index", "insert_batch", "select_neighbors",
    "try_rewire", "BucketMeta", "BuildParams", "CapacityError", "DimensionMismatchError", "GraphIndex",
    "RangePredicate", "SENTINEL", "SearchParams", "SearchResult", "SearchStats", "VectorRecord",
    "brute_force_arrays", "brute_force_search", "bucket_ids_of", "bucket_of", "create_index", "from_reference",
    "intersecting_buckets", "load_index", "save_index", "search", "search_arrays", "search_batch",
    "sq_distance", "sq_distances", "VectorStore", "partition_buckets", "gen_synthetic", "recall_at_k",
    "FvecsFormatError", "read_fvecs", "read_scalars", "write_fvecs", "write_scalars", "EvalReport",
    "GroundTruthCache", "SweepSpec", "run_sweep", "scc_count", "append_batch",
]
