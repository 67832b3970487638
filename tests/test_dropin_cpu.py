"""CPU checks of the drop-in surface: ``import bucketann`` through compat/ resolves
to this package with the reference's module layout, and the host-side value
types (VectorStore claim/publish, CandidateQueue, interleave_merge,
topk_ids_by_distance, derive_query_seed) behave like the reference's
(layout.py:22-79, searcher.py:52-87, builder.py:90-153). No device calls."""
import os
import subprocess
import sys
import threading

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bucketann_alias_resolves_every_reference_module():
    code = ("import bucketann, bucketann.core, bucketann.layout, bucketann.builder, bucketann.searcher, "
            "bucketann.updater, bucketann.evaluate, bucketann.dataio\n"
            "import paper_2604_16402_b200 as p\n"
            "assert bucketann is p and bucketann.layout is p.layout and bucketann.searcher is p.searcher\n"
            "from bucketann.layout import BucketMeta, VectorStore, append_batch, new_adjacency, partition_buckets\n"
            "from bucketann.builder import GlobalGraph, LocalGraphDraft, exact_knn_graph, fuse_remote_edges, "
            "interleave_merge, reinforce_reachability, topk_ids_by_distance\n"
            "from bucketann.searcher import CandidateQueue, derive_query_seed\n"
            "from bucketann.evaluate import generate_ranges, brute_force_search, recall_at_k\n"
            "from bucketann.dataio import gen_synthetic\n"
            "from bucketann import (BuildParams, BuildReport, BucketMeta, CapacityError, DimensionMismatchError,"
            " EvalReport, GraphIndex, GroundTruthCache, InsertReport, RangePredicate, SENTINEL, SearchParams,"
            " SearchResult, SweepSpec, VectorRecord, VectorStore, append_batch, brute_force_search, bucket_of,"
            " build_global_graph, build_index, build_local_phase, create_index, gen_synthetic, insert_batch,"
            " intersecting_buckets, load_index, partition_buckets, read_fvecs, read_scalars, recall_at_k,"
            " run_sweep, save_index, scc_count, search, search_batch, select_neighbors, sq_distance,"
            " sq_distances, try_rewire, write_fvecs, write_scalars)\n"
            "print('ok')\n")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.join(ROOT, "compat"), ROOT]))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.fixture(scope="module")
def g():
    import paper_2604_16402_b200 as g
    return g


def test_vector_store_claims_are_contiguous_and_count_publishes_in_order(g):
    st = g.VectorStore(4000, 4)
    meta = None
    starts = []
    lock = threading.Lock()

    def worker(i):
        b = np.full((37, 4), i, np.float32)
        iv = g.layout.append_batch(st, meta, b, np.full(37, 0.5, np.float32))
        with lock:
            starts.append(iv)

    th = [threading.Thread(target=worker, args=(i,)) for i in range(40)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    starts.sort()
    assert starts[0][0] == 0 and all(a[1] == b[0] for a, b in zip(starts, starts[1:]))
    assert st.count == 40 * 37
    # publish order: a later range completing first does not advance count
    s2 = g.VectorStore(10, 2)
    a, b = s2.claim(3), s2.claim(3)
    s2.publish(b, 3)
    assert s2.count == 0
    s2.publish(a, 3)
    assert s2.count == 6
    with pytest.raises(g.CapacityError):
        s2.claim(5)


def test_append_batch_validation_on_host_store(g):
    st = g.VectorStore(8, 3)
    with pytest.raises(g.DimensionMismatchError):
        g.layout.append_batch(st, None, np.zeros((2, 4), np.float32), np.zeros(2))
    with pytest.raises(ValueError):
        g.layout.append_batch(st, None, np.zeros((1, 3), np.float32), np.array([np.nan]))
    assert g.layout.append_batch(st, None, np.zeros((0, 3), np.float32), np.zeros(0)) == (0, 0)
    assert np.all(g.new_adjacency(5, 4) == g.SENTINEL) and g.new_adjacency(5, 4).dtype == np.uint32


def test_candidate_queue_matches_reference_semantics(g):
    q = g.CandidateQueue(4)
    q.admit(np.array([5, 3]), np.array([2.0, 1.0]))
    q.admit(np.array([9, 7, 8]), np.array([0.5, 1.0, 3.0]))
    assert list(q.slots) == [9, 3, 7, 5] and list(q.dists) == [0.5, 1.0, 1.0, 2.0]
    fr = q.frontier(2)
    assert list(fr) == [0, 1]
    q.expanded[fr] = True
    assert list(q.frontier(2)) == [2, 3]
    s, d = q.top_k(2)
    assert list(s) == [9, 3] and len(q) == 4


def test_builder_list_helpers(g):
    from paper_2604_16402_b200.builder import interleave_merge, topk_ids_by_distance
    assert interleave_merge([1, 2], [2, 3], 3) == [1, 2, 3]
    assert interleave_merge([1, 2], [2, 3], 2) == [1, 2]
    assert interleave_merge([], [5, 6], 4) == [5, 6]
    assert interleave_merge([7], [], 4) == [7]
    assert list(topk_ids_by_distance(np.array([[1.0, 0.5, 0.5, 0.5, 2.0]]), 2)[0]) == [1, 2]
    r = np.random.default_rng(0).random((6, 9))
    want = np.argsort(r, axis=1, kind="stable")[:, :4]
    assert np.array_equal(topk_ids_by_distance(r, 4), want)


def test_derive_query_seed_matches_seedsequence(g):
    for base, o in [(0, 0), (11, 3), (2 ** 64 - 1, 7), (5, 2 ** 31)]:
        want = int(np.random.SeedSequence([base, o]).generate_state(1, np.uint64)[0])
        assert g.derive_query_seed(base, o) == want


def test_insert_report_rewired_rows_behave_like_a_sorted_list():
    """InsertReport.rewired_rows (updater.py:42,261: sorted(rewired)) is returned as
    an array-backed sequence; every list use the reference and its tests make works."""
    from paper_2604_16402_b200.api import InsertReport, RowList
    rows = np.array([3, 7, 7000000, 2 ** 31 + 5], dtype=np.uint32)
    rl = RowList(rows)
    assert len(rl) == 4 and list(rl) == [3, 7, 7000000, 2 ** 31 + 5]
    assert rl == [3, 7, 7000000, 2 ** 31 + 5] and rl == (3, 7, 7000000, 2 ** 31 + 5)
    assert not (rl == [3, 7]) and rl != [3, 7, 7000000, 6]
    assert rl[0] == 3 and rl[-1] == 2 ** 31 + 5 and rl[1:3] == [7, 7000000]
    assert 7 in rl and 8 not in rl and set(rl) == {3, 7, 7000000, 2 ** 31 + 5}
    assert sorted(rl) == rl.tolist() and np.array_equal(np.asarray(rl), rows.astype(np.int64))
    assert {1, 3}.issubset(set(rl)) is False and {3, 7}.issubset(set(rl))
    rep = InsertReport(batch_size=2, rewired_rows=rl)
    assert rep.to_dict()["rewired_rows"] == [3, 7, 7000000, 2 ** 31 + 5]
    assert RowList(np.empty(0, np.uint32)) == [] and len(RowList(np.empty(0, np.uint32))) == 0


def test_search_batch_results_are_search_results():
    """search_batch's ResultList (api.py) against an eagerly built list: every item
    is a SearchResult whose slots / sq_dists / truncated / stats are the batch
    row's (searcher.py:34-49), including short (truncated) and empty rows."""
    import numpy as np
    from paper_2604_16402_b200.api import BatchResult, SearchResult, SearchStats
    nq, k = 7, 4
    names = ["iterations", "dist_evals", "seed_evals", "gathered", "in_range_new", "precheck_rejected",
             "seed_attempts", "expanded"]
    st = np.zeros(nq, dtype=[(f, "<u4") for f in names])
    for j, f in enumerate(names):
        st[f] = np.arange(nq) * 10 + j
    counts = np.array([4, 2, 0, 4, 1, 4, 3], np.uint32)
    slots = np.arange(nq * k, dtype=np.int64).reshape(nq, k)
    dists = slots.astype(np.float64) / 3
    rs = BatchResult(slots, dists, counts, st, 0.7).to_results(k)
    assert len(rs) == nq
    for i, r in enumerate(rs):
        c = int(counts[i])
        want = SearchResult(slots[i, :c], dists[i, :c], 0 < c < k,
                            SearchStats(*[int(st[f][i]) for f in names], elapsed_s=0.7 / nq))
        assert isinstance(r, SearchResult)
        assert np.array_equal(r.slots, want.slots) and np.array_equal(r.sq_dists, want.sq_dists)
        assert r.truncated == want.truncated and len(r) == c
        assert r.stats == want.stats
    assert rs[-1].stats.dist_evals == rs[6].stats.dist_evals == 61
    assert [len(r) for r in rs[1:4]] == [2, 0, 4]
    with pytest.raises(IndexError):
        rs[nq]
    nostats = BatchResult(slots, dists, counts, None, 0.7).to_results(k)
    assert nostats[0].stats == SearchStats(elapsed_s=0.7 / nq)
