"""Recall vs global pass at scale (cfg5-shaped rows): python tools/scale_check.py N [exact]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2604_16402_b200 as g  # noqa: E402
from paper_2604_16402_b200 import datasets as ds  # noqa: E402

n = int(sys.argv[1])
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["descent:3", "descent:8"]
X, S = ds.gen_lowrank(n, 96, seed=1000, w_seed=0)
Q = ds.lowrank_queries(2000, 96, seed=1)
lo, hi = ds.range_arrays(ds.generate_ranges(S, 0.1, 2000, 0))
for m in modes:
    parts = m.split(":")
    gp, r = parts[0], parts[1] if len(parts) > 1 else "3"
    kmax = int(parts[2]) if len(parts) > 2 else 32
    t0 = time.perf_counter()
    gi, rep = g.build_index(X, S, g.BuildParams(k_max=kmax, k_local=kmax // 2, bucket_capacity=10_000), global_pass=gp,
                            refine_rounds=int(r), k_g=min(kmax, 32))
    tb = time.perf_counter() - t0
    truth, _, tc = g.brute_force_arrays(gi, Q, lo, hi, 10)
    recs = []
    width = 2 if kmax > 32 else 4
    for itopk in (128, 224, 320, 512):
        rr = g.search_arrays(gi, Q, lo, hi, g.SearchParams(k=10, itopk=itopk, search_width=width, max_iterations=150),
                             seed_base=0)
        recs.append(round(ds.batch_recall(rr.slots, rr.counts, truth, tc, 10), 4))
    full = g.search_arrays(gi, Q, np.full(2000, -1.0), np.full(2000, 2.0), g.SearchParams(k=10, itopk=128, search_width=width), seed_base=0)
    ft, _, fc = g.brute_force_arrays(gi, Q, np.full(2000, -1.0), np.full(2000, 2.0), 10)
    print(f"n={n} {m}: build {tb:.1f} s (p1 {rep.phase1_seconds:.1f} p2 {rep.phase2_seconds:.1f}) "
          f"R@10 10%% itopk128/224/320/512 {recs}  full-range itopk128 "
          f"{ds.batch_recall(full.slots, full.counts, ft, fc, 10):.4f}", f"p2 detail: {rep.global_pass}", flush=True)
    del gi
