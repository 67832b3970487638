"""Build a config on the GPU and run the search kernel a few times (for ncu / timing).

    ncu --set full --profile-from-start off -k regex:k_search -c 1 -o gpurun_out/search \
        python tools/profile_search.py --config cfg2
    python tools/profile_search.py --config cfg2 --time        # QPS + recall per operating point
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2604_16402_b200 as g  # noqa: E402
from paper_2604_16402_b200 import datasets as ds  # noqa: E402

P = {"cfg1": (100_000, 128, 6250, 1000, 96, 4, 50), "cfg2": (1_000_000, 128, 10_000, 10_000, 256, 4, 100),
     "cfg3": (1_000_000, 960, 10_000, 10_000, 328, 4, 100)}
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--itopk", type=int)
ap.add_argument("--width", type=int)
ap.add_argument("--iters", type=int)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--time", action="store_true")
ap.add_argument("--points", default="")
ap.add_argument("--sel", type=float, default=0.1)
ap.add_argument("--nostats", action="store_true", help="profile the stats-free kernel instance")
a = ap.parse_args()
n, dim, cap, nq, itopk, width, iters = P[a.config]
itopk = a.itopk or itopk
width = a.width or width
iters = a.iters or iters
X, S = ds.gen_lowrank(n, dim, seed=0)
Q = ds.lowrank_queries(nq, dim, seed=1)
lo, hi = ds.range_arrays(ds.generate_ranges(S, a.sel, nq, 0))
gi, rep = g.build_index(X, S, g.BuildParams(k_max=32, k_local=16, bucket_capacity=cap))
points = [(itopk, width, iters)]
if a.points:
    points = [tuple(int(x) for x in p.split(":")) for p in a.points.split(",")]
truth = None
if a.time:
    import torch
    truth, _, tc = g.brute_force_arrays(gi, Q, lo, hi, 10)
    Qd, lod, hid = (torch.from_numpy(x).cuda() for x in (Q, lo, hi))
for it_, w_, mi_ in points:
    sp = g.SearchParams(k=10, itopk=it_, search_width=w_, max_iterations=mi_)
    if a.time:
        r = g.search_arrays(gi, Q, lo, hi, sp, seed_base=0)
        rec = ds.batch_recall(r.slots, r.counts, truth, tc, 10)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(a.reps):
            g.search_arrays(gi, Qd, lod, hid, sp, seed_base=0, stats=False)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / a.reps
        print(f"itopk {it_} width {w_} iters {mi_}: recall {rec:.4f} qps {nq / dt:,.0f} ({dt * 1e3:.2f} ms/batch)")
    else:
        import torch
        for rep_ in range(a.reps):
            if rep_ == a.reps - 1:  # ncu --profile-from-start off: only the last rep is captured
                torch.cuda.synchronize()
                torch.cuda.profiler.start()
            r = g.search_arrays(gi, Q, lo, hi, sp, seed_base=0, stats=not a.nostats)
            if rep_ == a.reps - 1:
                torch.cuda.synchronize()
                torch.cuda.profiler.stop()
        st = r.stats
        if st is not None:
            print("mean stats:", {f: float(np.mean(st[f])) for f in st.dtype.names})
