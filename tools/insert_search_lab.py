"""Time the insert's candidate search alone (full range, itopk = k = 128, width 4,
50 iterations) on the cfg2 index, repeatedly, on one stream, plus the same on
a fresh index each time -- to separate kernel variance from first-use costs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_16402_b200 as g  # noqa: E402
from paper_2604_16402_b200 import datasets as ds  # noqa: E402

X, S = ds.gen_lowrank(1_000_000, 128, seed=0)
Xi, _ = ds.gen_lowrank(100_000, 128, seed=2, w_seed=0)
Xd = torch.from_numpy(Xi).cuda()
params = g.BuildParams(k_max=32, k_local=16, bucket_capacity=10_000)
sp = g.SearchParams(k=128, itopk=128, search_width=4, max_iterations=50)
stream = torch.cuda.current_stream()
for rep in range(3):
    gi, _ = g.build_index(X, S, params)
    ts = [bench._event_ms(lambda: g.search_arrays(gi, Xd, 0.0, 1.0, sp, seed_base=0, stats=False), stream, 1)
          for _ in range(5)]
    print(f"index {rep}: candidate search ms {[round(t, 1) for t in ts]}", flush=True)
    del gi
