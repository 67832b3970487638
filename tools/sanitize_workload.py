"""Small end-to-end workload for compute-sanitizer (tests/test_gpu_sanitizer.py).

Touches every kernel family at sizes memcheck / racecheck finish in seconds:
partition, the device build (tcgen05 kNN screen + f64 rerank, exact global pass
and NN-descent, fuse, repair), search in bitmap and hash visited modes with and
without SearchStats, brute force, append, insert (candidates, forward
selection, rewiring, heal), the phase-level ABI (local / global / fuse /
reinforce), SCC, and the sharded pack + merge. Host numpy inputs only (no torch
import), so the sanitizer sees only libgrab's own CUDA work."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_16402_b200 as g  # noqa: E402
from paper_2604_16402_b200.datasets import gen_lowrank, lowrank_queries  # noqa: E402


def main():
    X, S = gen_lowrank(3000, 24, seed=0)
    params = g.BuildParams(k_max=16, k_local=8, bucket_capacity=400)
    g.partition_buckets(S, 400)
    gi, _ = g.build_index(X, S, params, capacity=4000)                      # exact global pass
    gd, _ = g.build_index(X, S, params, capacity=4000, global_pass="descent")  # NN-descent
    Q = lowrank_queries(64, 24, seed=1)
    rng = np.random.default_rng(0)
    lo = rng.random(64) * 0.8
    for width, stats in ((0.1, True), (0.1, False), (1.0, True)):        # bitmap / hash visited modes
        hi = np.minimum(lo + width, 1.0) if width < 1 else np.full(64, np.inf)
        l2 = lo if width < 1 else np.full(64, -np.inf)
        g.search_arrays(gi, Q, l2, hi, g.SearchParams(k=10, itopk=64), seed_base=3, stats=stats)
        g.brute_force_arrays(gi, Q, l2, hi, 10)
    g.search_arrays(gd, Q, lo, lo + 0.2, g.SearchParams(k=10, itopk=32, search_width=2), seed_base=1)
    Xn, Sn = gen_lowrank(400, 24, seed=2, w_seed=0)
    g.insert_batch(gi, Xn[:300], Sn[:300])
    g.append_batch(gi, None, Xn[300:], Sn[300:])
    g.scc_count(gi)
    # phase-level ABI on a host store
    st = g.VectorStore(1000, 24)
    meta = g.partition_buckets(S[:1000], 250, capacity=1000)
    g.append_batch(st, None, X[:1000], S[:1000])
    draft = g.build_local_phase(st, meta, params)
    gg = g.build_global_graph(st, params, k_g=16)
    adj = g.new_adjacency(1000, 16)
    g.fuse_remote_edges(draft, gg, st, meta, params, adj)
    g.reinforce_reachability(gi)
    # sharded route -> search -> pack -> exchange -> merge (one shard; both exchanges)
    if os.environ.get("SANITIZE_SHARD", "1") == "1":
        import torch
        from paper_2604_16402_b200 import shard as sh
        for ex in ("nccl", "p2p"):
            idx, _ = sh.ShardedIndex.build(X, S, np.arange(len(X), dtype=np.int64), params, rank=0, world=1,
                                           exchange=ex)
            idx.search(torch.from_numpy(Q).cuda(), lo, lo + 0.3, g.SearchParams(k=10, itopk=32), seed_base=0)
            torch.cuda.synchronize()
            idx.close_peers()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
