"""Times the host-buffer search path three ways at the cfg2 operating point:
pageable numpy, page-locked torch inputs, and the pinned result allocation alone."""
import time

import numpy as np
import torch

import paper_2604_16402_b200 as g
from paper_2604_16402_b200 import api, datasets as ds

n, dim, nq = 1_000_000, 128, 10_000
X, S = ds.gen_lowrank(n, dim, seed=0)
Q = ds.lowrank_queries(nq, dim, seed=1)
lo, hi = ds.range_arrays(ds.generate_ranges(S, 0.1, nq, 0))
gi, _ = g.build_index(X, S, g.BuildParams(k_max=32, k_local=16, bucket_capacity=10_000))
sp = g.SearchParams(k=10, itopk=296, search_width=4, max_iterations=100)
Qp, lop, hip = (torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (Q, lo, hi))


def t(fn, n=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


print("pageable ms", t(lambda: g.search_arrays(gi, Q, lo, hi, sp, seed_base=0)))
print("pinned zero-copy ms", t(lambda: g.search_arrays(gi, Qp, lop, hip, sp, seed_base=0)))
import os
os.environ["GRAB_NO_ZERO_COPY"] = "1"
print("pinned staged ms", t(lambda: g.search_arrays(gi, Qp, lop, hip, sp, seed_base=0)))
del os.environ["GRAB_NO_ZERO_COPY"]
print("pinned nostats ms", t(lambda: g.search_arrays(gi, Qp, lop, hip, sp, seed_base=0, stats=False)))
print("alloc4   ms", t(lambda: [api._pinned_empty((nq, 10), np.int64), api._pinned_empty((nq, 10), np.float64),
                                 api._pinned_empty(nq, np.uint32), api._pinned_empty(nq, g._lib.STATS_DTYPE)]))
Qd, lod, hid = Qp.cuda(), lop.cuda(), hip.cuda()
print("device   ms", t(lambda: g.search_arrays(gi, Qd, lod, hid, sp, seed_base=0)))
