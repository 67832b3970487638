"""Search-kernel lab: build a config's index once, then time k_search at given
operating points and selectivities (CUDA events, device-resident inputs).

    python tools/search_lab.py --config cfg2 --sels 0.01,0.1,0.5 --points 296:4:100,448:4:150 --reps 10

Prints one line per (selectivity, point, stats): ms per 10K batch, QPS, R@10,
and the algorithmic-bytes HBM fraction (bench.algorithmic_bytes)."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--sels", default="0.1")
    ap.add_argument("--points", default="296:4:100")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--nq", type=int)
    ap.add_argument("--pairs", help="sel@itopk:w:it,... (overrides --sels/--points)")
    a = ap.parse_args()
    import torch
    import bench
    import paper_2604_16402_b200 as g
    from paper_2604_16402_b200 import _lib, datasets as ds
    cfg = bench.PRESETS[a.config]
    n, dim, cap = cfg["n"], cfg["dim"], cfg["cap"]
    nq = a.nq or cfg["nq"]
    X, S = ds.gen_lowrank(n, dim, seed=0)
    gi, _ = g.build_index(X, S, g.BuildParams(k_max=32, k_local=16, bucket_capacity=cap))
    Q = ds.lowrank_queries(nq, dim, seed=1)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    Qd = torch.from_numpy(Q).to(dev)
    hbm, _ = bench.measured_peak_hbm()
    bench._gpu_warm(0, 0.5)
    if a.pairs:
        todo = [(float(p.split("@")[0]), [p.split("@")[1]]) for p in a.pairs.split(",")]
    else:
        todo = [(float(x), a.points.split(",")) for x in a.sels.split(",")]
    for sel, pts in todo:
        lo, hi = ds.range_arrays(ds.generate_ranges(S, sel, nq, 0))
        truth, _, tc = g.brute_force_arrays(gi, Q, lo, hi, 10)
        lod, hid = torch.from_numpy(lo).to(dev), torch.from_numpy(hi).to(dev)
        for pt in pts:
            itopk, w, it = (int(x) for x in pt.split(":"))
            sp = g.SearchParams(k=10, itopk=itopk, search_width=w, max_iterations=it)
            r = g.search_arrays(gi, Qd, lod, hid, sp, seed_base=0)
            rec = ds.batch_recall(r.slots.cpu().numpy(), r.counts.cpu().numpy(), truth, tc, 10)
            st = np.frombuffer(r.stats.cpu().numpy().astype(np.uint32).tobytes(), dtype=_lib.STATS_DTYPE)
            b = bench.algorithmic_bytes(st, (dim + 3) // 4 * 4, 32, 10)
            for stats in (False, True):
                ms = bench._event_ms(lambda: g.search_arrays(gi, Qd, lod, hid, sp, seed_base=0, stats=stats),
                                     stream, a.reps)
                print(f"sel={sel} pt={pt} stats={stats} ms={ms:.3f} qps={nq / ms * 1e3 / 1e6:.3f}M "
                      f"R@10={rec:.4f} frac={b / (ms / 1e3) / 1e9 / hbm:.3f}", flush=True)


if __name__ == "__main__":
    main()
