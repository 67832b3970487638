"""ctypes binding of libgrab.so (the C ABI declared in include/grab.h).

The product path has no CPU fallback: importing this module without the
built library, or calling into it without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .params import CapacityError, DimensionMismatchError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgrab.so")

OK, ERR_VALUE, ERR_DIMENSION, ERR_CAPACITY, ERR_CUDA, ERR_STATE = range(6)
MEM_HOST, MEM_DEVICE = 0, 1
SENTINEL = 0xFFFFFFFF
LIVE_ALL = 0xFFFFFFFFFFFFFFFF
ARR_X, ARR_SCALARS, ARR_ADJ, ARR_I2B, ARR_BOUNDARIES, ARR_B2I_OFFSETS, ARR_B2I_FLAT = range(7)
GRAPH_LOCAL_ONLY, GRAPH_GLOBAL_ONLY = 1, 2


class GrabDeviceError(RuntimeError):
    """A CUDA-side failure inside libgrab."""


class BuildParamsC(C.Structure):
    _fields_ = [("k_max", C.c_uint32), ("k_local", C.c_uint32), ("bucket_capacity", C.c_uint32),
                ("global_pass", C.c_uint32), ("proximal_fraction", C.c_double), ("proximal_window", C.c_double),
                ("alpha", C.c_double), ("rng_seed", C.c_uint64)]


class SearchParamsC(C.Structure):
    _fields_ = [("k", C.c_uint32), ("itopk", C.c_uint32), ("search_width", C.c_uint32),
                ("max_iterations", C.c_uint32), ("seed_count", C.c_uint32), ("_pad", C.c_uint32)]


STAT_FIELDS = ["iterations", "dist_evals", "seed_evals", "gathered", "in_range_new", "precheck_rejected",
               "seed_attempts", "expanded"]
STATS_DTYPE = np.dtype([(f, "<u4") for f in STAT_FIELDS])


class BuildReportC(C.Structure):
    _fields_ = [("n", C.c_uint64), ("m", C.c_uint32), ("isolated_nodes", C.c_uint32),
                ("phase1_seconds", C.c_double), ("phase2_seconds", C.c_double), ("fuse_seconds", C.c_double),
                ("total_seconds", C.c_double), ("cross_bucket_edge_ratio", C.c_double),
                ("global_descent", C.c_uint32), ("_pad", C.c_uint32)]


INSERT_FIELDS = ["batch_size", "bulk_built", "forward_accepted", "forward_rejected", "reverse_accepted",
                 "reverse_rejected", "evictions_necessary", "evictions_redundant", "forced_links", "n_rewired"]


class BuildDebugC(C.Structure):
    _fields_ = [("forward_rows", C.c_void_p), ("merged_rows", C.c_void_p), ("necessary", C.c_void_p),
                ("global_rows", C.c_void_p)]


class InsertReportC(C.Structure):
    _fields_ = [(f, C.c_uint64) for f in INSERT_FIELDS] + [("wall_time_s", C.c_double),
                                                          ("phase_seconds", C.c_double * 6)]


class InfoC(C.Structure):
    _fields_ = [("count", C.c_uint64), ("capacity", C.c_uint64), ("dim", C.c_uint32), ("k_max", C.c_uint32),
                ("k_local", C.c_uint32), ("m", C.c_uint32), ("built", C.c_int32), ("_pad", C.c_uint32),
                ("phys_capacity", C.c_uint64), ("device_bytes", C.c_uint64)]


P = C.c_void_p
u32, u64, i32, i64, dbl = C.c_uint32, C.c_uint64, C.c_int32, C.c_int64, C.c_double

_SIGS = {
    "grab_create": (C.c_int, [C.c_int, u32, u64, C.POINTER(BuildParamsC), C.POINTER(P)]),
    "grab_destroy": (None, [P]),
    "grab_last_error": (C.c_char_p, []),
    "grab_get_info": (C.c_int, [P, C.POINTER(InfoC)]),
    "grab_sync": (C.c_int, [P]),
    "grab_build": (C.c_int, [P, P, P, u64, C.c_int, u32, u32, u32, C.POINTER(BuildReportC)]),
    "grab_build_ex": (C.c_int, [P, P, P, u64, C.c_int, u32, u32, u32, C.POINTER(BuildReportC), P]),
    "grab_build_graph": (C.c_int, [P, u32, u32, u64, u32, C.POINTER(BuildReportC), P]),
    "grab_fuse": (C.c_int, [P, P, P, u32]),
    "grab_reinforce": (C.c_int, [P, C.POINTER(u64)]),
    "grab_insert": (C.c_int, [P, P, P, P, u64, u32, u32, C.POINTER(InsertReportC)]),
    "grab_last_rewired": (C.c_int, [P, P, u64, C.POINTER(u64)]),
    "grab_append": (C.c_int, [P, P, P, P, u64, u32, C.POINTER(u64), C.POINTER(u64)]),
    "grab_search": (C.c_int, [P, P, u64, P, P, u64, C.POINTER(SearchParamsC), P, u64, u64, u64, P, P, P, P, u32, P]),
    "grab_brute_force": (C.c_int, [P, P, u64, P, P, u64, u32, u64, P, P, P, u32, P]),
    "grab_bucket_select": (C.c_int, [P, P, P, u64, P, P, u32, P]),
    "grab_bucket_ids": (C.c_int, [P, P, u64, P, u32, P]),
    "grab_bucket_ids_raw": (C.c_int, [P, u32, P, u64, P]),
    "grab_partition": (C.c_int, [C.c_int, P, u64, u32, C.c_int, P, u32, C.POINTER(u32), P, u32, P]),
    "grab_bucket_select_raw": (C.c_int, [P, u32, P, P, u64, P, P]),
    "grab_sq_distances": (C.c_int, [P, P, u64, u32, P]),
    "grab_import": (C.c_int, [P, u64, P, P, P, P, u32, P, P, P]),
    "grab_read": (C.c_int, [P, C.c_int, u64, u64, P]),
    "grab_select_neighbors": (C.c_int, [P, u64, u32, i64, P, P, P, u32, u32, dbl, P, P]),
    "grab_try_rewire": (C.c_int, [P, u64, u32, P, u32, u32, u32, dbl, dbl, u32, P, P]),
    "grab_shard_pack": (C.c_int, [u64, P, P, P, P, u32, u32, u32, P, P, P]),
    "grab_merge_topk": (C.c_int, [u32, u32, u32, u32, P, P, P, P, P, P]),
    "grab_shard_pack_p2p": (C.c_int, [u64, P, P, P, P, u32, u32, u32, u32, P, P, P]),
    "grab_reverse_merge_raw": (C.c_int, [C.c_int, P, u64, u32, P, u32, u32, P]),
    "grab_shard_sync_bytes": (u64, [u32]),
    "grab_shard_pack_p2p_sync": (C.c_int, [u32, u64, P, P, P, P, u32, u32, u32, u32, P, P, P, P, u64, P, P]),
    "grab_merge_topk_p2p": (C.c_int, [u32, u32, u32, u32, P, P, P, P, P, u32, P, P, u64, P]),
    "grab_ipc_alloc": (C.c_int, [u64, C.POINTER(P), P]),
    "grab_ipc_open": (C.c_int, [P, C.POINTER(P)]),
    "grab_ipc_close": (C.c_int, [P]),
    "grab_ipc_free": (C.c_int, [P]),
    "grab_derive_seeds": (C.c_int, [u64, P, u64, P]),
    "grab_scc_count": (C.c_int, [P, u64, P]),
    "grab_scc_count_raw": (C.c_int, [P, u64, u32, u64, P]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libgrab.so not found at {LIB_PATH}; build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = (lib.grab_last_error() or b"").decode()
    if rc == ERR_CAPACITY:
        raise CapacityError(msg)
    if rc == ERR_DIMENSION:
        raise DimensionMismatchError(msg)
    if rc == ERR_VALUE:
        raise ValueError(msg)
    if rc == ERR_STATE:
        raise RuntimeError(msg)
    raise GrabDeviceError(msg)


def ptr(a) -> int | None:
    """Address of a numpy array / torch tensor (None passes NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    raise TypeError(type(a))
