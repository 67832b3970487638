"""Pin the CPU oracle (oracle/) against golden vectors frozen from the live reference.

Goldens: tests/golden/make_golden.py (run with the reference on PYTHONPATH).
"""
import numpy as np
import pytest

from oracle import beam, construct, index_state as ist, ingest, rng as R

STAT_KEYS = ["iterations", "dist_evals", "seed_evals", "gathered", "in_range_new",
             "precheck_rejected", "seed_attempts"]
GRID = [dict(k=10, itopk=128, search_width=4, max_iterations=50),
        dict(k=10, itopk=32, search_width=1, max_iterations=50),
        dict(k=5, itopk=64, search_width=2, max_iterations=10),
        dict(k=16, itopk=256, search_width=4, max_iterations=100)]


def test_rng_restatement_matches_reference_draws(golden):
    g = golden("rng")
    for (b, o), want in zip(g["pairs"].tolist(), g["derived"].tolist()):
        assert R.derive_query_seed(int(b), int(o)) == want
        assert beam.derive_seed(int(b), int(o)) == want
    for i, s in enumerate(g["seeds"].tolist()):
        for j, t in enumerate(g["totals"].tolist()):
            assert R.PCG64(int(s)).integers(int(t), 128) == g["draws"][i, j].tolist()


def test_partition_and_lookup(golden):
    g = golden("layout")
    cases = {
        "uniform": (np.random.default_rng(0).random(10_000, dtype=np.float32), 1000, "quantile"),
        "skewed": ((np.random.default_rng(3).random(5000, dtype=np.float32) ** 8).astype(np.float32), 500, "quantile"),
        "equal": (np.full(100, 5.0, np.float32), 10, "quantile"),
        "width": (np.random.default_rng(2).random(1000, dtype=np.float32), 100, "width"),
        "ties": (np.round(np.random.default_rng(4).random(3000) * 20).astype(np.float32), 97, "quantile"),
        "odd": (np.random.default_rng(5).standard_normal(1237).astype(np.float32), 100, "quantile"),
    }
    for name, (s, cap, strat) in cases.items():
        e = ist.partition_edges(s, cap, strat)
        assert e.tobytes() == g[f"{name}_boundaries"].tobytes(), name
        assert np.array_equal(ist.bucket_lookup(e, s), g[f"{name}_i2b"][: len(s)]), name
    b = g["iv_boundaries"]
    got = [ist.bucket_interval(b, lo, hi) for lo, hi in zip(g["iv_lower"], g["iv_upper"])]
    assert np.array_equal(np.array(got), g["iv_lohi"])
    assert np.array_equal(ist.bucket_lookup(b, g["bid_scalars"]), g["bid_ids"])


def _check_search_cases(idx, Q, S, prefix, g, nq):
    n = idx.count
    for si, sel in enumerate([0.01, 0.1, 0.5, 1.0]):
        ranges = beam.window_ranges(S[:n], sel, nq, 7)
        assert np.array_equal(np.array(ranges)[:, 0], g[f"{prefix}_sel{si}_lower"])
        for gi, p in enumerate(GRID):
            for i, (q, (lo, hi)) in enumerate(zip(Q, ranges)):
                cfg = ist.SearchCfg(lower=lo, upper=hi, rng_seed=beam.derive_seed(11, i), **p)
                r = beam.beam_search(idx, q, cfg)
                key = f"{prefix}_sel{si}_g{gi}_"
                c = g[key + "counts"][i]
                assert len(r.slots) == c
                assert np.array_equal(r.slots, g[key + "slots"][i, :c]), (si, gi, i)
                assert np.array_equal(r.sq_dists, g[key + "dists"][i, :c])
                assert r.truncated == g[key + "truncated"][i]
                assert [getattr(r.stats, k) for k in STAT_KEYS] == g[key + "stats"][i].tolist()
        for i, (q, (lo, hi)) in enumerate(zip(Q, ranges)):
            s_, d_ = beam.exact_filtered(idx, q, 10, lo, hi)
            assert np.array_equal(s_, g[f"{prefix}_sel{si}_bf_slots"][i, : len(s_)])
            assert np.array_equal(d_, g[f"{prefix}_sel{si}_bf_dists"][i, : len(s_)])
    res = beam.beam_search_batch(idx, Q, ist.SearchCfg(k=10, lower=0.2, upper=0.45, itopk=64, rng_seed=21))
    for i, r in enumerate(res):
        c = g[f"{prefix}_batch_counts"][i]
        assert np.array_equal(r.slots, g[f"{prefix}_batch_slots"][i, :c])


def test_small_build_is_byte_identical(golden):
    g = golden("small")
    V, S = ist.gen_synthetic(2000, 8, "clusters", rng_seed=1)
    cfg = ist.BuildCfg(k_max=16, k_local=8, bucket_capacity=250)
    idx, draft, G = construct.build(V, S, cfg)
    assert np.array_equal(draft.forward, g["draft_forward"])
    assert np.array_equal(draft.merged, g["draft_rows"])
    assert np.array_equal(draft.necessary, g["draft_necessary"])
    assert np.array_equal(G, g["global_rows"])
    assert ist.container_bytes(idx) == g["container"].tobytes()
    assert construct.cross_ratio(idx) == pytest.approx(float(g["cross_ratio"]), abs=0)


def test_small_search_matches_reference(golden):
    g = golden("small")
    idx = ist.index_from_container(g["container"].tobytes(), ist.BuildCfg(k_max=16, k_local=8, bucket_capacity=250))
    V, S = ist.gen_synthetic(2000, 8, "clusters", rng_seed=1)
    Q, _ = ist.gen_synthetic(64, 8, "clusters", rng_seed=1)
    Q = Q + np.float32(0.01)
    _check_search_cases(idx, Q, S, "s", g, 64)
    srt = np.sort(S)
    edges = [(2.0, 3.0), (float(srt[0]), float(srt[2])), (-np.inf, np.inf), (float(srt[0]), float(srt[-1]))]
    for i, (lo, hi) in enumerate(edges):
        r = beam.beam_search(idx, V[0], ist.SearchCfg(k=10, lower=lo, upper=hi, itopk=64, rng_seed=5))
        c = g["edge_counts"][i]
        assert np.array_equal(r.slots, g["edge_slots"][i, :c])
        assert r.truncated == g["edge_truncated"][i]


def test_mid_search_matches_reference(golden):
    g = golden("mid")
    idx = ist.index_from_container(g["container"].tobytes())
    V, S = ist.gen_synthetic(10_000 + 120, 16, "clusters", rng_seed=2)
    _check_search_cases(idx, V[10_000:10_048], S[:10_000], "m", g, 48)


def test_descent_matches_reference(golden):
    g = golden("descent")
    r = np.random.default_rng(9)
    V = r.standard_normal((2000, 16)).astype(np.float32)
    S = r.random(2000, dtype=np.float32)
    idx = ist.empty_index(16, 2000, ist.BuildCfg())
    ist.append_rows(idx, V, S, with_meta=False)
    assert np.array_equal(construct.global_pass(idx, k_g=32, refine_rounds=3, exact_limit=0), g["rows"])
    assert np.array_equal(construct.global_pass(idx, k_g=8, refine_rounds=0, exact_limit=0), g["rows0"])


def test_insert_matches_reference(golden):
    g = golden("insert")
    V, S = ist.gen_synthetic(3500, 12, rng_seed=5)
    cfg = ist.BuildCfg(k_max=16, k_local=8, bucket_capacity=600, alpha=0.6)
    idx, _, _ = construct.build(V[:3000], S[:3000], cfg)
    assert np.array_equal(idx.adjacency[:3000], g["base_adj"])
    t = ingest.insert(idx, V[3000:], S[3000:])
    keys = ["batch_size", "bulk_built", "forward_accepted", "forward_rejected", "reverse_accepted",
            "reverse_rejected", "evictions_necessary", "evictions_redundant", "forced_links"]
    assert [getattr(t, k) for k in keys] == g["report"].tolist()
    assert t.rewired_rows == g["rewired"].tolist()
    assert np.array_equal(idx.adjacency[:3500], g["adj"])
    V2, S2 = ist.gen_synthetic(300, 12, rng_seed=55)
    t2 = ingest.insert(idx, V2, S2)
    assert [getattr(t2, k) for k in keys] == g["report2"].tolist()
    assert np.array_equal(idx.adjacency[:3800], g["adj2"])
    V3, S3 = ist.gen_synthetic(1200, 8, rng_seed=7)
    idx3 = ist.empty_index(8, 2400, ist.BuildCfg(k_max=8, k_local=4, bucket_capacity=500))
    t3 = ingest.insert(idx3, V3, S3)
    assert [getattr(t3, k) for k in keys] == g["report3"].tolist()
    assert np.array_equal(idx3.adjacency[:1200], g["adj3"])
