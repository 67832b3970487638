"""Time build_index on a config several times in one process (phase split).

    python tools/build_lab.py --config cfg2 --reps 3
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_16402_b200 as g  # noqa: E402
from paper_2604_16402_b200 import datasets as ds  # noqa: E402

P = {"cfg1": (100_000, 128, 6250), "cfg2": (1_000_000, 128, 10_000), "cfg3": (1_000_000, 960, 10_000)}
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--warm-rows", type=int, default=0, help="untimed build of this many rows first")
ap.add_argument("--reserve-gb", type=float, default=0, help="grow the default memory pool by this much first")
a = ap.parse_args()
n, dim, cap = P[a.config]
X, S = ds.gen_lowrank(n, dim, seed=0)
x = torch.randn(4096, 4096, device="cuda")
for _ in range(50):  # clock ramp
    x = x @ x
    x /= x.norm()
torch.cuda.synchronize()
if a.reserve_gb:
    from cuda.bindings import runtime as rt
    g.create_index(dim, 16, g.BuildParams(k_max=32, k_local=16, bucket_capacity=cap))  # sets the pool threshold
    t0 = time.perf_counter()
    err, p = rt.cudaMallocAsync(int(a.reserve_gb * 2**30), 0)
    rt.cudaFreeAsync(p, 0)
    rt.cudaStreamSynchronize(0)
    print(f"pool reserve {a.reserve_gb} GB: {time.perf_counter() - t0:.3f} s ({err})", flush=True)
if a.warm_rows:
    t0 = time.perf_counter()
    gw, _ = g.build_index(X[:a.warm_rows], S[:a.warm_rows], g.BuildParams(k_max=32, k_local=16, bucket_capacity=cap))
    torch.cuda.synchronize()
    del gw
    print(f"warm build {a.warm_rows}: {time.perf_counter() - t0:.3f} s", flush=True)
for r in range(a.reps):
    t0 = time.perf_counter()
    gi, rep = g.build_index(X, S, g.BuildParams(k_max=32, k_local=16, bucket_capacity=cap))
    torch.cuda.synchronize()
    print(f"rep {r}: wall {time.perf_counter() - t0:.3f} s  lib total {rep.total_seconds:.3f}  phase1 {rep.phase1_seconds:.3f}  "
          f"phase2 {rep.phase2_seconds:.3f}  fuse {rep.fuse_seconds:.3f}", flush=True)
    del gi
