"""Does clock sampling perturb the timed search loop? (cfg2, itopk 296)"""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_16402_b200 as g  # noqa: E402
from paper_2604_16402_b200 import datasets as ds  # noqa: E402

X, S = ds.gen_lowrank(1_000_000, 128, seed=0)
Q = ds.lowrank_queries(10_000, 128, seed=1)
lo, hi = ds.range_arrays(ds.generate_ranges(S, 0.1, 10_000, 0))
gi, _ = g.build_index(X, S, g.BuildParams(bucket_capacity=10_000))
Qd, lod, hid = (torch.from_numpy(x).cuda() for x in (Q, lo, hi))
sp = g.SearchParams(k=10, itopk=296, search_width=4, max_iterations=100)
st = torch.cuda.current_stream()


def timed(n=20):
    for _ in range(3):
        g.search_arrays(gi, Qd, lod, hid, sp, seed_base=0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(n):
        g.search_arrays(gi, Qd, lod, hid, sp, seed_base=0)
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for rep in range(2):
    print("none        ", round(timed(), 3), flush=True)
    with bench.ClockSampler(0) as c:
        print("pynvml 20ms ", round(timed(), 3), c.summary()["samples"], flush=True)
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks_event_reasons.active", "--format=csv",
                          "-lms", "200"], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    time.sleep(1.0)
    print("smi -lms 200", round(timed(), 3), flush=True)
    p.terminate()
    p.wait()
