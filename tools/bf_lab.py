"""Time the exact filtered brute force on cfg2 (10K queries at 1 / 10 / 50 %):
the tensor-core path (default) and the SIMT scan (GRAB_BF_SIMT=1), device-resident
inputs, CUDA events; checks the two agree bit for bit."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_16402_b200 as g  # noqa: E402
from paper_2604_16402_b200 import datasets as ds  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n, dim, cap = (bench.PRESETS[cfg][k] for k in ("n", "dim", "cap"))
X, S = ds.gen_lowrank(n, dim, seed=0)
Q = ds.lowrank_queries(10_000, dim, seed=1)
gi, _ = g.build_index(X, S, g.BuildParams(k_max=32, k_local=16, bucket_capacity=cap))
stream = torch.cuda.current_stream()
for sel in (0.01, 0.1, 0.5):
    lo, hi = ds.range_arrays(ds.generate_ranges(S, sel, 10_000, 0))
    out = {}
    for mode in ("tc", "simt"):
        if mode == "simt":
            os.environ["GRAB_BF_SIMT"] = "1"
        ms = bench._event_ms(lambda: g.brute_force_arrays(gi, Q, lo, hi, 10), stream, 3)
        out[mode] = g.brute_force_arrays(gi, Q, lo, hi, 10)
        os.environ.pop("GRAB_BF_SIMT", None)
        print(f"{cfg} sel {sel} {mode}: {ms:.2f} ms per 10K queries (host arrays)", flush=True)
    if os.environ.get("BF_PROFILE"):  # ncu --profile-from-start off: one tensor-core call
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        g.brute_force_arrays(gi, Q, lo, hi, 10)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    same = all(np.array_equal(a, b, equal_nan=True) for a, b in zip(out["tc"], out["simt"]))
    print(f"  identical: {same}", flush=True)
