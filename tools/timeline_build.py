"""Live per-kernel time of one cfg2 build (torch.profiler / CUPTI), summed by kernel name."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2604_16402_b200 as g  # noqa: E402
from paper_2604_16402_b200 import datasets as ds  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n, dim, cap = (bench.PRESETS[cfg][k] for k in ("n", "dim", "cap"))
X, S = ds.gen_lowrank(n, dim, seed=0)
params = g.BuildParams(k_max=32, k_local=16, bucket_capacity=cap)
g.build_index(X, S, params)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    gi, rep = g.build_index(X, S, params)
    torch.cuda.synchronize()
agg = collections.Counter()
cnt = collections.Counter()
for e in prof.events():
    if e.device_type.name == "CUDA":
        agg[e.name[:70]] += e.device_time
        cnt[e.name[:70]] += 1
tot = sum(agg.values())
print(f"total device time {tot / 1e3:.1f} ms; lib total {rep.total_seconds * 1e3:.1f} ms")
for k, v in agg.most_common(20):
    print(f"{v / 1e3:8.2f} ms x{cnt[k]:3d}  {k}")
