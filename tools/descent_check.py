"""GPU NN-descent vs the reference goldens (tests/golden/descent.npz) and exact-vs-descent builds."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2604_16402_b200 as g  # noqa: E402
from paper_2604_16402_b200 import datasets as ds  # noqa: E402

gd = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "descent.npz"))
r = np.random.default_rng(9)
V = r.standard_normal((2000, 16)).astype(np.float32)
S = r.random(2000, dtype=np.float32)
for kg, rounds, key in ((8, 0, "rows0"), (32, 3, "rows")):
    _, _, dr = g.build_index(V, S, g.BuildParams(), k_g=kg, refine_rounds=rounds, return_draft=True,
                             global_pass="descent")
    want = gd[key]
    same_rows = np.mean([np.array_equal(dr.global_rows[i], want[i]) for i in range(len(want))])
    same_sets = np.mean([set(dr.global_rows[i]) == set(want[i]) for i in range(len(want))])
    overlap = np.mean([len(set(dr.global_rows[i]) & set(want[i])) / kg for i in range(len(want))])
    print(f"{key}: rows identical {same_rows:.4f} sets identical {same_sets:.4f} overlap {overlap:.4f}", flush=True)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300_000
X, S = ds.gen_lowrank(n, 128, seed=0)
Q = ds.lowrank_queries(2000, 128, seed=1)
lo, hi = ds.range_arrays(ds.generate_ranges(S, 0.1, 2000, 0))
for gp in ("exact", "descent"):
    t0 = time.perf_counter()
    gi, rep = g.build_index(X, S, g.BuildParams(bucket_capacity=10_000), global_pass=gp)
    tb = time.perf_counter() - t0
    truth, _, tc = g.brute_force_arrays(gi, Q, lo, hi, 10)
    recs = []
    for itopk in (64, 128, 224):
        rr = g.search_arrays(gi, Q, lo, hi, g.SearchParams(k=10, itopk=itopk, max_iterations=100), seed_base=0)
        recs.append(round(ds.batch_recall(rr.slots, rr.counts, truth, tc, 10), 4))
    print(f"n={n} {gp}: build {tb:.2f} s (phase2 {rep.phase2_seconds:.2f} s, pass={rep.global_pass}) "
          f"recall@itopk64/128/224 {recs}", flush=True)
