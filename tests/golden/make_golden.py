"""Freeze golden vectors from the LIVE reference package.

Run in the build container (the reference exists only there):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every array written here is an output of ``bucketann`` itself (numpy 2.3.5),
never of this repo's oracle or kernels. Inputs are regenerated from seeds by
the tests (``bucketann.gen_synthetic`` draw order, restated in
oracle/index_state.py), so the fixtures hold outputs only.
"""
from __future__ import annotations

import io
import os
import sys

import numpy as np

import bucketann as ba
from bucketann import builder as bb
from bucketann.evaluate import generate_ranges
from bucketann.searcher import derive_query_seed
from bucketann.layout import bucket_ids_of

OUT = os.path.dirname(os.path.abspath(__file__))
STAT_KEYS = ["iterations", "dist_evals", "seed_evals", "gathered", "in_range_new",
             "precheck_rejected", "seed_attempts"]


def pack_results(results, k):
    nq = len(results)
    slots = np.full((nq, k), -1, np.int64)
    dists = np.full((nq, k), np.nan, np.float64)
    counts = np.zeros(nq, np.int32)
    trunc = np.zeros(nq, bool)
    stats = np.zeros((nq, len(STAT_KEYS)), np.int64)
    for i, r in enumerate(results):
        counts[i] = len(r.slots)
        slots[i, : len(r.slots)] = r.slots
        dists[i, : len(r.slots)] = r.sq_dists
        trunc[i] = r.truncated
        stats[i] = [getattr(r.stats, key) for key in STAT_KEYS]
    return dict(slots=slots, dists=dists, counts=counts, truncated=trunc, stats=stats)


def container(index):
    buf = io.BytesIO()
    path = os.path.join(OUT, "_tmp.grab")
    ba.save_index(index, path)
    raw = open(path, "rb").read()
    os.remove(path)
    return np.frombuffer(raw, dtype=np.uint8)


def rng_golden():
    r = np.random.default_rng(12345)
    bases = [0, 1, 7, 21, 2**32 - 1, 2**32, 2**40 + 5, 2**64 - 1] + [int(x) for x in r.integers(0, 2**63, 8)]
    ords = [0, 1, 5, 1000, 2**31, 2**32 + 3]
    pairs = np.array([(b, o) for b in bases for o in ords], dtype=np.uint64)
    derived = np.array([derive_query_seed(int(b), int(o)) for b, o in pairs], dtype=np.uint64)
    seeds = [0, 3, 9, int(derived[5]), int(derived[17]), 2**63 + 11]
    totals = [1, 2, 3, 17, 250, 6250, 100000, 2**31 + 11, 2**32 - 1]
    draws = np.zeros((len(seeds), len(totals), 128), np.int64)
    for i, s in enumerate(seeds):
        for j, t in enumerate(totals):
            draws[i, j] = np.random.default_rng(s).integers(0, t, size=128)
    np.savez_compressed(os.path.join(OUT, "rng.npz"), pairs=pairs, derived=derived,
                        seeds=np.array(seeds, np.uint64), totals=np.array(totals, np.int64), draws=draws)


def layout_golden():
    out = {}
    cases = {
        "uniform": (np.random.default_rng(0).random(10_000, dtype=np.float32), 1000, "quantile"),
        "skewed": ((np.random.default_rng(3).random(5000, dtype=np.float32) ** 8).astype(np.float32), 500, "quantile"),
        "equal": (np.full(100, 5.0, np.float32), 10, "quantile"),
        "width": (np.random.default_rng(2).random(1000, dtype=np.float32), 100, "width"),
        "ties": (np.round(np.random.default_rng(4).random(3000) * 20).astype(np.float32), 97, "quantile"),
        "odd": (np.random.default_rng(5).standard_normal(1237).astype(np.float32), 100, "quantile"),
    }
    for name, (s, cap, strat) in cases.items():
        meta = ba.partition_buckets(s, cap, strategy=strat)
        out[f"{name}_boundaries"] = meta.boundaries
        out[f"{name}_i2b"] = meta.index_to_bucket
    # bucket interval lookups on equal-width and quantile edges
    r = np.random.default_rng(9)
    lows = r.uniform(-0.5, 1.5, 400)
    widths = r.uniform(0, 1, 400)
    meta = ba.partition_buckets(cases["uniform"][0], 1000)
    out["iv_boundaries"] = meta.boundaries
    out["iv_lower"] = lows
    out["iv_upper"] = lows + widths
    out["iv_lohi"] = np.array([ba.intersecting_buckets(meta, ba.RangePredicate(a, b))
                               for a, b in zip(lows, lows + widths)], np.int32)
    s = r.uniform(-0.2, 1.2, 500).astype(np.float32)
    out["bid_scalars"] = s
    out["bid_ids"] = bucket_ids_of(meta, s)
    np.savez_compressed(os.path.join(OUT, "layout.npz"), **out)


def search_cases(index, X_queries, scalars, prefix, out):
    """A grid of ranges/params; single-query search with explicit seeds and batch search."""
    n = index.count
    nq = len(X_queries)
    sels = [0.01, 0.1, 0.5, 1.0]
    grid = [dict(k=10, itopk=128, search_width=4, max_iterations=50),
            dict(k=10, itopk=32, search_width=1, max_iterations=50),
            dict(k=5, itopk=64, search_width=2, max_iterations=10),
            dict(k=16, itopk=256, search_width=4, max_iterations=100)]
    for si, sel in enumerate(sels):
        ranges = generate_ranges(scalars[:n], sel, nq, 7)
        out[f"{prefix}_sel{si}_lower"] = np.array([r.lower for r in ranges])
        out[f"{prefix}_sel{si}_upper"] = np.array([r.upper for r in ranges])
        for gi, g in enumerate(grid):
            res = [ba.search(index, q, ba.SearchParams(range=r, rng_seed=derive_query_seed(11, i), **g))
                   for i, (q, r) in enumerate(zip(X_queries, ranges))]
            for key, val in pack_results(res, g["k"]).items():
                out[f"{prefix}_sel{si}_g{gi}_{key}"] = val
        # exact oracle
        bf = [ba.brute_force_search(index.store, q, 10, r) for q, r in zip(X_queries, ranges)]
        slots = np.full((nq, 10), -1, np.int64)
        dists = np.full((nq, 10), np.nan)
        for i, (s_, d_) in enumerate(bf):
            slots[i, : len(s_)] = s_
            dists[i, : len(s_)] = d_
        out[f"{prefix}_sel{si}_bf_slots"] = slots
        out[f"{prefix}_sel{si}_bf_dists"] = dists
    # search_batch with one shared range and derived seeds
    rr = ba.RangePredicate(0.2, 0.45)
    res = ba.search_batch(index, X_queries, ba.SearchParams(k=10, range=rr, itopk=64, rng_seed=21))
    for key, val in pack_results(res, 10).items():
        out[f"{prefix}_batch_{key}"] = val


def small_golden():
    """small_index fixture of the reference tests (test_search.py:20-25) + pieces."""
    V, S = ba.gen_synthetic(2000, 8, "clusters", rng_seed=1)
    params = ba.BuildParams(k_max=16, k_local=8, bucket_capacity=250)
    index, rep = ba.build_index(V, S, params)
    out = {"container": container(index), "cross_ratio": rep.cross_bucket_edge_ratio,
           "isolated": rep.isolated_nodes, "bucket_sizes": np.array(rep.bucket_sizes)}
    draft = ba.build_local_phase(index.store, index.meta, params)
    out["draft_forward"] = draft.forward_rows
    out["draft_rows"] = draft.rows
    out["draft_necessary"] = draft.necessary_counts
    out["global_rows"] = ba.build_global_graph(index.store, params).rows
    Q, _ = ba.gen_synthetic(64, 8, "clusters", rng_seed=1)
    Q = Q + np.float32(0.01)
    search_cases(index, Q, S, "s", out)
    # edge cases: empty range, tiny range, unbounded, exact hit
    srt = np.sort(S)
    edge = []
    for (lo, hi) in [(2.0, 3.0), (float(srt[0]), float(srt[2])), (-np.inf, np.inf), (float(srt[0]), float(srt[-1]))]:
        r = ba.search(index, V[0], ba.SearchParams(k=10, range=ba.RangePredicate(lo, hi), itopk=64, rng_seed=5))
        edge.append(r)
    for key, val in pack_results(edge, 10).items():
        out[f"edge_{key}"] = val
    np.savez_compressed(os.path.join(OUT, "small.npz"), **out)


def mid_golden():
    """mid_index fixture (test_search.py:28-33): 10k x 16 clusters, 120 held-out queries."""
    V, S = ba.gen_synthetic(10_000 + 120, 16, "clusters", rng_seed=2)
    params = ba.BuildParams(k_max=32, k_local=16, bucket_capacity=1000)
    index, rep = ba.build_index(V[:10_000], S[:10_000], params)
    out = {"container": container(index), "cross_ratio": rep.cross_bucket_edge_ratio}
    search_cases(index, V[10_000:10_000 + 48], S[:10_000], "m", out)
    np.savez_compressed(os.path.join(OUT, "mid.npz"), **out)


def descent_golden():
    """NN-descent global pass (test_builder.py:118-129 shape, exact_limit=0)."""
    r = np.random.default_rng(9)
    V = r.standard_normal((2000, 16)).astype(np.float32)
    S = r.random(2000, dtype=np.float32)
    store = ba.VectorStore(2000, 16)
    ba.append_batch(store, None, V, S)
    gg = ba.build_global_graph(store, ba.BuildParams(), k_g=32, refine_rounds=3, exact_limit=0)
    gg0 = ba.build_global_graph(store, ba.BuildParams(), k_g=8, refine_rounds=0, exact_limit=0)
    np.savez_compressed(os.path.join(OUT, "descent.npz"), rows=gg.rows, rows0=gg0.rows)


def insert_golden():
    """Insert into a built index (test_updater.py:175-184 shape) and empty-index bulk build."""
    out = {}
    V, S = ba.gen_synthetic(3000 + 500, 12, rng_seed=5)
    params = ba.BuildParams(k_max=16, k_local=8, bucket_capacity=600, alpha=0.6)
    index, _ = ba.build_index(V[:3000], S[:3000], params)
    out["base_adj"] = index.adjacency[:3000].copy()
    rep = ba.insert_batch(index, V[3000:], S[3000:])
    out["adj"] = index.adjacency[:3500].copy()
    keys = ["batch_size", "bulk_built", "forward_accepted", "forward_rejected", "reverse_accepted",
            "reverse_rejected", "evictions_necessary", "evictions_redundant", "forced_links"]
    out["report"] = np.array([getattr(rep, k) for k in keys], np.int64)
    out["rewired"] = np.array(rep.rewired_rows, np.int64)
    # second batch into the grown index
    V2, S2 = ba.gen_synthetic(300, 12, rng_seed=55)
    rep2 = ba.insert_batch(index, V2, S2)
    out["adj2"] = index.adjacency[:3800].copy()
    out["report2"] = np.array([getattr(rep2, k) for k in keys], np.int64)
    # empty-index bulk build (test_updater.py:198-207)
    V3, S3 = ba.gen_synthetic(1200, 8, rng_seed=7)
    idx3 = ba.create_index(8, 2400, ba.BuildParams(k_max=8, k_local=4, bucket_capacity=500))
    rep3 = ba.insert_batch(idx3, V3, S3)
    out["adj3"] = idx3.adjacency[:1200].copy()
    out["report3"] = np.array([getattr(rep3, k) for k in keys], np.int64)
    np.savez_compressed(os.path.join(OUT, "insert.npz"), **out)


def sweep_golden():
    """run_sweep over the small_index fixture (evaluate.py:249-307): the
    deterministic columns of every grid row, the CSV header, and the GTC1
    ground-truth files the disk cache wrote (name = SHA-256 key, bytes)."""
    import tempfile
    from bucketann import evaluate as ev
    V, S = ba.gen_synthetic(2000, 8, "clusters", rng_seed=1)
    index, _ = ba.build_index(V, S, ba.BuildParams(k_max=16, k_local=8, bucket_capacity=250))
    Q, _ = ba.gen_synthetic(64, 8, "clusters", rng_seed=1)
    Q = Q + np.float32(0.01)
    spec = ev.SweepSpec(selectivities=[0.01, 0.1, 0.5, 1.0], itopk_values=[32, 64], search_widths=[1, 4],
                        max_iterations_values=[10, 50], query_count=48, rng_seed=3)
    out = {}
    with tempfile.TemporaryDirectory() as d:
        rep = ev.run_sweep(index, Q, spec, gt_cache=ev.GroundTruthCache(d))
        rep.write_csv(os.path.join(d, "sweep.csv"))
        out["csv_header"] = np.frombuffer(open(os.path.join(d, "sweep.csv"), "rb").readline(), np.uint8)
        names = sorted(f for f in os.listdir(d) if f.endswith(".gt"))
        out["gt_names"] = np.array(names)
        for i, f in enumerate(names):
            out[f"gt_{i}"] = np.frombuffer(open(os.path.join(d, f), "rb").read(), np.uint8)
    cols = ["selectivity", "k", "itopk", "search_width", "max_iterations", "recall", "dist_evals_per_query", "scc"]
    out["cols"] = np.array(cols)
    out["rows"] = np.array([[row[c] for c in cols] for row in rep.rows], np.float64)
    np.savez_compressed(os.path.join(OUT, "sweep.npz"), **out)


ALL = ["rng_golden", "layout_golden", "small_golden", "mid_golden", "descent_golden", "insert_golden",
       "sweep_golden"]

if __name__ == "__main__":
    assert "bucketann" in sys.modules
    for name in (sys.argv[1:] or ALL):
        globals()[name]()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))
