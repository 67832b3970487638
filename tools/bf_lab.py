"""Time the exact filtered brute force (k_bruteforce) on cfg2: 10K queries at 10 %."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_16402_b200 as g  # noqa: E402
from paper_2604_16402_b200 import datasets as ds  # noqa: E402

X, S = ds.gen_lowrank(1_000_000, 128, seed=0)
Q = ds.lowrank_queries(10_000, 128, seed=1)
lo, hi = ds.range_arrays(ds.generate_ranges(S, 0.1, 10_000, 0))
gi, _ = g.build_index(X, S, g.BuildParams(k_max=32, k_local=16, bucket_capacity=10_000))
Qd, lod, hid = (torch.from_numpy(a).cuda() for a in (Q, lo, hi))
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s, d, c = g.brute_force_arrays(gi, Q, lo, hi, 10)
    torch.cuda.synchronize()
    print(f"brute force 10K queries: {(time.perf_counter() - t0) * 1e3:.1f} ms (host arrays)", flush=True)
print("checksum", int(s[:, 0].sum()), float(d[:, 0].sum()))
