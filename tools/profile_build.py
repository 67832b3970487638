"""Build a config twice; the second build runs under torch.cuda.profiler (for
ncu --profile-from-start off, e.g. -k regex:k_knn_screen_tc -c 1 or
-k regex:k_descent)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_16402_b200 as g  # noqa: E402
from paper_2604_16402_b200 import datasets as ds  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n, dim, cap = (bench.PRESETS[cfg][k] for k in ("n", "dim", "cap"))
X, S = ds.gen_lowrank(n, dim, seed=0)
params = g.BuildParams(k_max=32, k_local=16, bucket_capacity=cap)
g.build_index(X, S, params)
torch.cuda.synchronize()
torch.cuda.profiler.start()
gi, rep = g.build_index(X, S, params)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(rep.to_dict())
