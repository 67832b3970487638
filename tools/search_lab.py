"""Search timing lab: build cfg once, then time operating points several ways.

    python tools/search_lab.py --config cfg2 --points 224:4:100 --reps 20
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_16402_b200 as g  # noqa: E402
from paper_2604_16402_b200 import datasets as ds  # noqa: E402

P = {"cfg1": (100_000, 128, 6250, 1000), "cfg2": (1_000_000, 128, 10_000, 10_000),
     "cfg3": (1_000_000, 960, 10_000, 10_000)}
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--points", default="224:4:100")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--sel", type=float, default=0.1)
ap.add_argument("--n", type=int)
a = ap.parse_args()
n, dim, cap, nq = P[a.config]
n = a.n or n
X, S = ds.gen_lowrank(n, dim, seed=0)
Q = ds.lowrank_queries(nq, dim, seed=1)
lo, hi = ds.range_arrays(ds.generate_ranges(S, a.sel, nq, 0))
t0 = time.perf_counter()
gi, rep = g.build_index(X, S, g.BuildParams(k_max=32, k_local=16, bucket_capacity=cap))
print(f"build {time.perf_counter() - t0:.2f} s", flush=True)
truth, _, tc = g.brute_force_arrays(gi, Q, lo, hi, 10)
Qd, lod, hid = (torch.from_numpy(x).cuda() for x in (Q, lo, hi))
st = torch.cuda.current_stream()
for p in a.points.split(","):
    it_, w_, mi_ = (int(x) for x in p.split(":"))
    sp = g.SearchParams(k=10, itopk=it_, search_width=w_, max_iterations=mi_)
    r = g.search_arrays(gi, Q, lo, hi, sp, seed_base=0)
    rec = ds.batch_recall(r.slots, r.counts, truth, tc, 10)
    s = r.stats
    means = {f: round(float(np.mean(s[f])), 1) for f in s.dtype.names}
    for stats in (False, True):
        for _ in range(3):
            g.search_arrays(gi, Qd, lod, hid, sp, seed_base=0, stats=stats)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(a.reps):
            g.search_arrays(gi, Qd, lod, hid, sp, seed_base=0, stats=stats)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        print(f"{p} stats={stats}: recall {rec:.4f} {ms:.3f} ms/batch  qps {nq / ms * 1e3:,.0f}", flush=True)
    print("   ", means, flush=True)
