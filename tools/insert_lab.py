"""Time insert_batch on cfg2 (100K into a 1M build, device-resident batch):
Python wall, the library's own wall_time_s and its phase split.

    python tools/insert_lab.py [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_16402_b200 as g  # noqa: E402
from paper_2604_16402_b200 import datasets as ds  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
X, S = ds.gen_lowrank(1_000_000, 128, seed=0)
Xi, Si = ds.gen_lowrank(100_000, 128, seed=2, w_seed=0)
Xd, Sd = torch.from_numpy(Xi).cuda(), torch.from_numpy(Si).cuda()
params = g.BuildParams(k_max=32, k_local=16, bucket_capacity=10_000)
gw, _ = g.build_index(X[:200_000], S[:200_000], params)
g.insert_batch(gw, Xd[:20_000], Sd[:20_000])  # warm-up (modules, pools)
del gw
for r in range(reps):
    gi, _ = g.build_index(X, S, params)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = g.insert_batch(gi, Xd, Sd)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ph = {k: round(v * 1e3, 2) for k, v in rep.phase_seconds.items()}
    print(f"rep {r}: wall {wall * 1e3:.1f} ms ({len(Xi) / wall / 1e6:.3f} M vectors/s), library {rep.wall_time_s * 1e3:.1f} "
          f"ms, phases ms {ph}, rewired {len(rep.rewired_rows)}", flush=True)
    del gi
