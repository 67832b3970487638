import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2604_16402_b200 as g
from paper_2604_16402_b200 import datasets as ds
X, S = ds.gen_lowrank(100_000, 128, seed=0)
gi, _ = g.build_index(X, S, g.BuildParams(k_max=32, k_local=16, bucket_capacity=6250))
Q = ds.lowrank_queries(2000, 128, seed=1)
sp = g.SearchParams(k=10, itopk=96, search_width=4, max_iterations=50)
for sel in (0.01, 0.9, 0.01, 0.9, 0.01, 0.9):
    lo, hi = ds.range_arrays(ds.generate_ranges(S, sel, len(Q), 0))
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        g.search_arrays(gi, Q, lo, hi, sp, seed_base=0, stats=False)
        torch.cuda.synchronize(); print(sel, rep, round((time.perf_counter() - t0) * 1e3, 2), 'ms', flush=True)
