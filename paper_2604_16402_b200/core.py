"""``bucketann.core`` surface (reference core.py:1-147): value types, errors and
the f64-accumulated squared-L2 distance (computed on the device with the same
reduction tree as the search / brute-force kernels)."""
from __future__ import annotations

from .api import sq_distance, sq_distances
from .params import (BuildParams, CapacityError, DimensionMismatchError, RangePredicate, SearchParams,
                     VectorRecord)

__all__ = ["BuildParams", "CapacityError", "DimensionMismatchError", "RangePredicate", "SearchParams",
           "VectorRecord", "sq_distance", "sq_distances"]
