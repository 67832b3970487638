"""Rows wider than 1024 floats (embedding-style d = 1536): build (streamed-A
tcgen05 screen), search, brute force and insert give the oracle's results."""
import numpy as np
import pytest

from oracle import beam, construct, index_state as ist, ingest

pytestmark = pytest.mark.gpu
KEYS = ["batch_size", "bulk_built", "forward_accepted", "forward_rejected", "reverse_accepted", "reverse_rejected",
        "evictions_necessary", "evictions_redundant", "forced_links"]
STAT_KEYS = ["iterations", "dist_evals", "seed_evals", "gathered", "in_range_new", "precheck_rejected",
             "seed_attempts"]


@pytest.fixture(scope="module")
def g():
    import paper_2604_16402_b200 as g
    return g


def test_d1536_search_brute_force_insert_match_oracle(g):
    d = 1536
    X, S = ist.gen_lowrank(2_300, d, seed=41)
    cfg = ist.BuildCfg(k_max=16, k_local=8, bucket_capacity=500)
    ref, _, _ = construct.build(X[:2_000], S[:2_000], cfg, capacity=2_400)
    gi = g.load_index(ist.container_bytes(ref), g.BuildParams(k_max=16, k_local=8, bucket_capacity=500))
    Q = ist.lowrank_queries(8, d, seed=42)
    for lo, hi in ((0.1, 0.6), (-1.0, 2.0)):
        p = g.SearchParams(k=10, itopk=64, search_width=4, max_iterations=40)
        res = g.search_arrays(gi, Q, lo, hi, p, seed_base=4)
        s, dd, c = g.brute_force_arrays(gi, Q, lo, hi, 10)
        for i in range(len(Q)):
            want = beam.beam_search(ref, Q[i], ist.SearchCfg(k=10, lower=lo, upper=hi, itopk=64, search_width=4,
                                                             max_iterations=40, rng_seed=beam.derive_seed(4, i)))
            n = int(res.counts[i])
            assert np.array_equal(res.slots[i, :n], want.slots)
            assert [int(res.stats[i][f]) for f in STAT_KEYS] == [getattr(want.stats, f) for f in STAT_KEYS]
            ws, _ = beam.exact_filtered(ref, Q[i], 10, lo, hi)
            assert np.array_equal(s[i, : int(c[i])], ws)
    rep = g.insert_batch(gi, X[2_000:], S[2_000:])
    t = ingest.insert(ref, X[2_000:], S[2_000:])
    assert [getattr(rep, k) for k in KEYS] == [getattr(t, k) for k in KEYS]
    assert np.array_equal(gi.adjacency[:2_300], ref.adjacency[:2_300])


def test_d1536_device_build_pass1_exact(g):
    r = np.random.default_rng(43)
    V = r.standard_normal((600, 1536)).astype(np.float32)
    S = r.random(600, dtype=np.float32)
    gi, rep, dr = g.build_index(V, S, g.BuildParams(k_max=16, k_local=8, bucket_capacity=600), return_draft=True)
    X = V.astype(np.float64)
    dm = ((X[:, None, :] - X[None, :, :]) ** 2).sum(-1)
    np.fill_diagonal(dm, np.inf)
    want = np.array([np.lexsort((np.arange(600), dm[i]))[:16] for i in range(600)])
    assert np.array_equal(dr.forward_rows.astype(np.int64), want)
    with pytest.raises(ValueError):  # d > 2048 is rejected, not served by a fallback
        g.build_index(r.standard_normal((64, 2_100)).astype(np.float32), r.random(64, dtype=np.float32),
                      g.BuildParams(k_max=8, k_local=4, bucket_capacity=64))
