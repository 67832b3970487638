"""Freeze BASELINE-shape goldens (configs[0], "cfg1") from the LIVE reference.

Run in the build container (the reference exists only there). The build and
search goldens (cfg1.npz) take ~3 min; the reference's insert runs at a few
vectors/s at this size, so the inserts (cfg1_insert.npz) take hours:

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden_cfg1.py

Workload (BASELINE.json configs[0]): 100 000 x 128 low-rank-16
vectors (``datasets.gen_lowrank(100_000, 128, seed=0)``), uniform scalars,
bucket_capacity 6 250 (m = 16), k = 10. Everything written is an output of
``bucketann`` itself (numpy 2.3.5):

* the reference-built graph: adjacency rows [0, n), boundaries, M_I2B
  (``builder.build_index``, builder.py:503-548) -- X and S are regenerated from
  the seed by the tests, so only the graph is stored;
* ``search`` (searcher.py:156-233) outputs -- slots, f64 distances, truncated
  and all 7 SearchStats counters -- for 256 queries at 1 %, 10 % and 50 %
  selectivity and two operating points (itopk 128 / 50 iterations, itopk 296 /
  100 iterations, width 4), with per-query seeds derive_query_seed(11, i);
* the cfg1 workload proper: 1 000 queries at 10 % with default SearchParams and
  the exact filtered brute force (evaluate.py:22-44) -> the reference's
  recall@10 on its own graph;
* 20 000 inserted vectors (``gen_lowrank(20_000, 128, seed=2, w_seed=0)``) as
  four 5 000-vector ``insert_batch`` calls (updater.py:154-263) into that graph,
  in cfg1_insert.npz: each batch's InsertReport counters and sorted rewired
  rows, and a 64-bit hash of every adjacency row [0, 100K + inserted) after the
  last batch done (the file is rewritten per batch; ``ins_batches`` says how many).
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

import bucketann as ba
from bucketann.evaluate import generate_ranges
from bucketann.searcher import derive_query_seed

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from paper_2604_16402_b200.datasets import gen_lowrank, lowrank_queries  # noqa: E402  (pure numpy generators)

from make_golden import STAT_KEYS, pack_results  # noqa: E402

N, D, CAP = 100_000, 128, 6_250
N_INS = 20_000
INS_BATCHES = 4
SELS = [0.01, 0.1, 0.5]
GRID = [dict(k=10, itopk=128, search_width=4, max_iterations=50),
        dict(k=10, itopk=296, search_width=4, max_iterations=100)]
INSERT_KEYS = ["batch_size", "bulk_built", "forward_accepted", "forward_rejected", "reverse_accepted",
               "reverse_rejected", "evictions_necessary", "evictions_redundant", "forced_links"]


def row_hash(adj: np.ndarray) -> np.ndarray:
    """Polynomial hash of every u32 row (wrapping u64 arithmetic); tests restate it."""
    p = np.uint64(0x9E3779B97F4A7C15)
    pw = np.ones(adj.shape[1], np.uint64)
    with np.errstate(over="ignore"):  # wrapping u64 arithmetic is the point
        for j in range(1, adj.shape[1]):
            pw[j] = pw[j - 1] * p
        return (adj.astype(np.uint64) * pw[None, :]).sum(axis=1, dtype=np.uint64)


def main():
    out = {}
    X, S = gen_lowrank(N, D, seed=0)
    params = ba.BuildParams(bucket_capacity=CAP)
    t0 = time.time()
    index, rep = ba.build_index(X, S, params, n_threads=os.cpu_count() or 1)
    print(f"build {time.time() - t0:.1f}s m={index.meta.m}", flush=True)
    out["adj"] = index.adjacency[:N].copy()
    out["boundaries"] = index.meta.boundaries.copy()
    out["i2b"] = index.meta.index_to_bucket[:N].astype(np.uint8)
    out["build_report"] = np.array([rep.m, rep.isolated_nodes], np.int64)
    out["cross_ratio"] = rep.cross_bucket_edge_ratio
    out["build_seconds"] = rep.total_seconds

    Q = lowrank_queries(256, D, seed=1)
    t0 = time.time()
    for si, sel in enumerate(SELS):
        ranges = generate_ranges(S, sel, len(Q), 7)
        out[f"sel{si}_lower"] = np.array([r.lower for r in ranges])
        out[f"sel{si}_upper"] = np.array([r.upper for r in ranges])
        for gi, g in enumerate(GRID):
            res = [ba.search(index, q, ba.SearchParams(range=r, rng_seed=derive_query_seed(11, i), **g))
                   for i, (q, r) in enumerate(zip(Q, ranges))]
            for key, val in pack_results(res, g["k"]).items():
                out[f"sel{si}_g{gi}_{key}"] = val
        bf = [ba.brute_force_search(index.store, q, 10, r) for q, r in zip(Q, ranges)]
        slots = np.full((len(Q), 10), -1, np.int64)
        for i, (s_, _) in enumerate(bf):
            slots[i, : len(s_)] = s_
        out[f"sel{si}_bf_slots"] = slots
    print(f"search grid {time.time() - t0:.1f}s", flush=True)

    # cfg1 workload: 1K queries at 10 %, default SearchParams, batch seeds (searcher.py:236-248)
    Q1 = lowrank_queries(1000, D, seed=1)
    ranges = generate_ranges(S, 0.1, len(Q1), 0)
    res = [ba.search(index, q, ba.SearchParams(range=r, rng_seed=derive_query_seed(0, i)))
           for i, (q, r) in enumerate(zip(Q1, ranges))]
    packed = pack_results(res, 10)
    out["w_slots"] = packed["slots"]
    out["w_counts"] = packed["counts"]
    rec = []
    for r_, q, rg in zip(res, Q1, ranges):
        ts, _ = ba.brute_force_search(index.store, q, 10, rg)
        rec.append(ba.recall_at_k(r_.slots, ts, 10))
    out["w_recall"] = float(np.nanmean(rec))
    print(f"cfg1 workload recall {out['w_recall']:.4f}", flush=True)

    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), **out)
    print("cfg1.npz", os.path.getsize(os.path.join(HERE, "cfg1.npz")), flush=True)

    # 20K inserted rows as INS_BATCHES append-only batches into the reference-built
    # graph; cfg1_insert.npz is rewritten after every batch (ins_batches = batches done)
    Vn, Sn = gen_lowrank(N_INS, D, seed=2, w_seed=0)
    ins = {}
    per = N_INS // INS_BATCHES
    for b in range(INS_BATCHES):
        t0 = time.time()
        irep = ba.insert_batch(index, Vn[b * per:(b + 1) * per], Sn[b * per:(b + 1) * per])
        print(f"insert batch {b}: {time.time() - t0:.1f}s", flush=True)
        ins[f"ins{b}_report"] = np.array([getattr(irep, k) for k in INSERT_KEYS], np.int64)
        ins[f"ins{b}_rewired"] = np.array(sorted(irep.rewired_rows), np.uint32)
        ins[f"ins{b}_seconds"] = irep.wall_time_s
        ins["ins_batches"] = b + 1
        ins["ins_row_hash"] = row_hash(index.adjacency[: N + (b + 1) * per])
        np.savez_compressed(os.path.join(HERE, "cfg1_insert.npz"), **ins)


if __name__ == "__main__":
    assert len(STAT_KEYS) == 7
    main()
