import sys, time, os
sys.path.insert(0, "/root/repo")
import torch
torch.cuda.set_device(0)
import paper_2604_16402_b200 as g
from paper_2604_16402_b200 import datasets as ds
X, S = ds.gen_lowrank(1_000_000, 128, seed=0)
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    gi, rep = g.build_index(X, S, g.BuildParams(bucket_capacity=10_000))
    torch.cuda.synchronize()
    print(i, f"wall {time.perf_counter()-t0:.3f}", {k: round(v, 3) for k, v in rep.to_dict().items() if 'seconds' in k}, flush=True)
    del gi
