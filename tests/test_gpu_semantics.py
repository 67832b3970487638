"""Reference search / insert semantics on the device, mirroring the reference's
own tests (test_search.py, test_updater.py) on a GPU-built index: exact hits,
full range == unfiltered, batch == serial with derived seeds, batch edge sizes,
truncation, counter economy, recall monotone in the queue size, every newcomer
reachable after an insert, capacity errors."""
import numpy as np
import pytest

from oracle import beam, index_state as ist

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    import paper_2604_16402_b200 as g
    return g


@pytest.fixture(scope="module")
def built(g):
    X, S = ist.gen_lowrank(20_000, 32, seed=31)
    gi, _ = g.build_index(X, S, g.BuildParams(k_max=32, k_local=16, bucket_capacity=2_000))
    return gi, X, S


def test_exact_hit_returns_stored_slot(g, built):  # test_search.py exact hit
    gi, X, S = built
    for i in (0, 17, 4_321, 19_999):
        p = g.SearchParams(k=5, range=g.RangePredicate(float(S[i]) - 0.01, float(S[i]) + 0.01), itopk=64)
        r = g.search(gi, X[i], p)
        assert r.slots[0] == i and r.sq_dists[0] == 0.0


def test_full_range_equivalent_to_unfiltered(g, built):
    gi, X, S = built
    Q = ist.lowrank_queries(16, 32, seed=32)
    p = g.SearchParams(k=10, itopk=96)
    a = g.search_arrays(gi, Q, -np.inf, np.inf, p, seed_base=3)
    b = g.search_arrays(gi, Q, float(S.min()), float(S.max()), p, seed_base=3)
    assert np.array_equal(a.slots, b.slots) and np.array_equal(a.counts, b.counts)


def test_batch_matches_serial_with_derived_seeds(g, built):
    gi, X, S = built
    Q = ist.lowrank_queries(12, 32, seed=33)
    p = g.SearchParams(k=10, range=g.RangePredicate(0.2, 0.45), itopk=64, rng_seed=9)
    batch = g.search_batch(gi, Q, p)
    for i, q in enumerate(Q):
        pi = g.SearchParams(k=10, range=g.RangePredicate(0.2, 0.45), itopk=64, rng_seed=beam.derive_seed(9, i))
        one = g.search(gi, q, pi)
        assert np.array_equal(one.slots, batch[i].slots) and np.array_equal(one.sq_dists, batch[i].sq_dists)
        assert one.stats.dist_evals == batch[i].stats.dist_evals


@pytest.mark.parametrize("nq", [0, 1, 31, 32, 33, 257])
def test_batch_edge_sizes(g, built, nq):
    gi, X, S = built
    Q = ist.lowrank_queries(max(nq, 1), 32, seed=34)[:nq]
    out = g.search_batch(gi, Q, g.SearchParams(k=10, range=g.RangePredicate(0.1, 0.3), itopk=64))
    assert len(out) == nq
    assert all(len(r.slots) == 10 and np.all(np.diff(r.sq_dists) >= 0) for r in out)


def test_truncated_flag_when_fewer_valid_than_k(g, built):
    gi, X, S = built
    srt = np.sort(S)
    lo, hi = float(srt[100]), float(srt[105])  # exactly 6 rows in range
    r = g.search(gi, X[0], g.SearchParams(k=10, range=g.RangePredicate(lo, hi), itopk=64))
    inr = np.nonzero((S >= np.float32(lo)) & (S <= np.float32(hi)))[0]
    assert 0 < len(r.slots) == len(inr) < 10 and r.truncated
    assert set(r.slots.tolist()) == set(inr.tolist())


def test_precheck_economy_counters(g, built):
    gi, X, S = built
    Q = ist.lowrank_queries(64, 32, seed=35)
    r = g.search_arrays(gi, Q, 0.3, 0.4, g.SearchParams(k=10, itopk=128), seed_base=1)
    st = r.stats
    assert np.all(st["dist_evals"] == st["seed_evals"] + st["in_range_new"])
    assert np.all(st["precheck_rejected"] + st["in_range_new"] <= st["gathered"])
    assert np.all(st["iterations"] <= 50) and np.all(st["seed_attempts"] >= st["seed_evals"])


def test_recall_monotone_in_queue_size(g, built):
    gi, X, S = built
    Q = ist.lowrank_queries(200, 32, seed=36)
    from paper_2604_16402_b200 import datasets as ds
    rs = beam.window_ranges(S, 0.1, len(Q), 2)
    lo = np.array([a for a, _ in rs])
    hi = np.array([b for _, b in rs])
    ts, _, tc = g.brute_force_arrays(gi, Q, lo, hi, 10)
    rec = []
    for it in (16, 32, 64, 128, 256):
        r = g.search_arrays(gi, Q, lo, hi, g.SearchParams(k=10, itopk=it, max_iterations=100), seed_base=5)
        rec.append(ds.batch_recall(r.slots, r.counts, ts, tc, 10))
    assert all(b >= a - 0.01 for a, b in zip(rec, rec[1:])), rec
    assert rec[-1] >= 0.95, rec


def test_insert_every_newcomer_reachable_and_capacity_error(g):
    X, S = ist.gen_lowrank(6_600, 16, seed=37)
    gi, _ = g.build_index(X[:6_000], S[:6_000], g.BuildParams(k_max=16, k_local=8, bucket_capacity=1_000),
                          capacity=6_700)
    g.insert_batch(gi, X[6_000:6_600], S[6_000:6_600])
    A = gi.adjacency[:6_600]
    indeg = np.zeros(6_600, np.int64)
    valid = A[A != np.uint32(0xFFFFFFFF)].astype(np.int64)
    np.add.at(indeg, valid, 1)
    assert (indeg[6_000:] > 0).all()  # _heal_unreachable guarantee (updater.py:266-324)
    with pytest.raises(g.CapacityError):
        g.insert_batch(gi, X[:200], S[:200])
    assert gi.count == 6_600


@pytest.mark.parametrize("shared", [False, True])
def test_work_order_does_not_change_results(g, built, shared):
    """Batches of >= 2048 queries are claimed in a work order (per-query ranges:
    by lower bound, k_order_by_lower; one shared range: by LSH cell,
    k_sim_project / k_order_by_cell -- csrc/search.cu). Every query's search is
    independent of the order: the batch equals the same queries run in
    512-query chunks (below the threshold: claimed in index order) with the same
    per-query seeds -- slots, f64 distances, counts and every counter."""
    gi, X, S = built
    nq = 3000
    Q = ist.lowrank_queries(nq, 32, seed=33)
    if shared:
        lo, hi = np.float64(0.2), np.float64(0.7)
    else:
        r = beam.window_ranges(S, 0.1, nq, 9)
        lo = np.array([a for a, _ in r])
        hi = np.array([b for _, b in r])
        # unbounded ranges go through the ordering kernel too (its end bins)
        lo[:40:2] = -np.inf
        hi[1:40:2] = np.inf
    p = g.SearchParams(k=10, itopk=96)
    whole = g.search_arrays(gi, Q, lo, hi, p, seed_base=5)
    for c0 in range(0, nq, 512):
        sl = slice(c0, min(nq, c0 + 512))
        part = g.search_arrays(gi, Q[sl], lo if shared else lo[sl], hi if shared else hi[sl], p, seed_base=5,
                               ordinal0=c0)
        assert np.array_equal(part.slots, whole.slots[sl])
        assert np.array_equal(part.dists, whole.dists[sl], equal_nan=True)
        assert np.array_equal(part.counts, whole.counts[sl])
        assert np.array_equal(part.stats, whole.stats[sl])


def test_work_order_with_invalid_device_bounds(g, built):
    """Device-resident bounds skip the host's lower <= upper check: inverted and
    NaN ranges reach the ordering kernel and the search kernel, which give those
    queries an empty result; every other query of the (ordered) batch returns
    what it returns alone."""
    import torch
    gi, X, S = built
    nq = 2500
    Q = ist.lowrank_queries(nq, 32, seed=34)
    r = beam.window_ranges(S, 0.1, nq, 10)
    lo = np.array([a for a, _ in r])
    hi = np.array([b for _, b in r])
    bad = np.zeros(nq, bool)
    bad[5:200:7] = True
    lo[5:200:14], hi[5:200:14] = hi[5:200:14], lo[5:200:14]  # inverted
    lo[12:200:14] = np.nan
    seeds = (np.arange(nq, dtype=np.uint64) * np.uint64(7919) + np.uint64(5))
    p = g.SearchParams(k=10, itopk=96)
    dev = torch.device("cuda", gi.device)
    res = g.search_arrays(gi, torch.from_numpy(Q).to(dev), torch.from_numpy(lo).to(dev),
                          torch.from_numpy(hi).to(dev), p, seeds=torch.from_numpy(seeds.view(np.int64)).to(dev))
    counts = res.counts.cpu().numpy()
    assert (counts[bad] == 0).all()
    good = ~bad
    alone = g.search_arrays(gi, Q[good], lo[good], hi[good], p, seeds=seeds[good])
    assert np.array_equal(res.slots.cpu().numpy()[good], alone.slots)
    assert np.array_equal(counts[good], alone.counts)
