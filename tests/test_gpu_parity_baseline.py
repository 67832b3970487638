"""GPU parity at a BASELINE shape: configs[0] ("cfg1", 100 000 x 128 low-rank-16,
bucket_capacity 6 250 -> m = 16, k = 10), against goldens frozen from the LIVE
reference by tests/golden/make_golden_cfg1.py.

d = 128 is the headline dimension: these tests run the ``k_search<NC=1, EPL=4,
FULL=true, STATS>`` instances (both STATS values) and the d = 128 brute force
that produce every bench number, on the reference's own graph:

* search (searcher.py:156-233): identical slots, f64 distances (rtol 1e-12),
  truncated flags and all 7 SearchStats counters, at 1 / 10 / 50 % selectivity
  and two operating points; host, page-locked (zero-copy) and device-resident
  buffers agree;
* brute force (evaluate.py:22-44): identical IDs;
* the cfg1 workload (1K queries at 10 %, default SearchParams, batch seeds):
  identical slots and the reference's own recall@10;
* build (builder.py:503-548): the GPU-built graph's recall@10 within 0.005 of
  the reference-built graph's (north_star), on 10K queries per selectivity;
* insert (updater.py:154-263): 20K rows as four 5K batches into the reference
  graph -- every InsertReport, rewired-row set and adjacency row [0, 120K) as
  the reference left them (cfg1_insert.npz); and GPU build + GPU insert vs
  reference build + insert within 0.005 recall.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N, D, CAP, N_INS = 100_000, 128, 6_250, 20_000
SELS = [0.01, 0.1, 0.5]
GRID = [dict(k=10, itopk=128, search_width=4, max_iterations=50),
        dict(k=10, itopk=296, search_width=4, max_iterations=100)]
STAT_KEYS = ["iterations", "dist_evals", "seed_evals", "gathered", "in_range_new", "precheck_rejected",
             "seed_attempts"]
INSERT_KEYS = ["batch_size", "bulk_built", "forward_accepted", "forward_rejected", "reverse_accepted",
               "reverse_rejected", "evictions_necessary", "evictions_redundant", "forced_links"]
RECALL_TOL = 0.005  # north_star: GPU-built / inserted recall within 0.005 of the reference's


def row_hash(adj: np.ndarray) -> np.ndarray:
    """make_golden_cfg1.row_hash restated: wrapping u64 polynomial over each row."""
    p = np.uint64(0x9E3779B97F4A7C15)
    pw = np.ones(adj.shape[1], np.uint64)
    with np.errstate(over="ignore"):  # wrapping u64 arithmetic is the point
        for j in range(1, adj.shape[1]):
            pw[j] = pw[j - 1] * p
        return (adj.astype(np.uint64) * pw[None, :]).sum(axis=1, dtype=np.uint64)


@pytest.fixture(scope="module")
def g():
    import paper_2604_16402_b200 as g
    return g


@pytest.fixture(scope="module")
def data():
    from paper_2604_16402_b200.datasets import gen_lowrank, lowrank_queries
    X, S = gen_lowrank(N, D, seed=0)
    Vn, Sn = gen_lowrank(N_INS, D, seed=2, w_seed=0)
    return dict(X=X, S=S, Vn=Vn, Sn=Sn, Q=lowrank_queries(256, D, seed=1), Q1=lowrank_queries(1000, D, seed=1),
                Qr=lowrank_queries(10_000, D, seed=5))


@pytest.fixture(scope="module")
def gold(golden):
    return golden("cfg1")


INS_BATCHES = 4  # make_golden_cfg1.py: 20K inserts as four append-only batches


def ref_graph(g, data, gold):
    """The reference-built graph in the device layout (capacity 2n like build_index)."""
    from paper_2604_16402_b200.graph import import_state
    i2b = gold["i2b"].astype(np.int32)
    order = np.argsort(i2b, kind="stable")
    cuts = np.searchsorted(i2b[order], np.arange(len(gold["boundaries"])))
    lists = [order[cuts[b]:cuts[b + 1]] for b in range(len(cuts) - 1)]
    gi = g.create_index(D, 2 * N, g.BuildParams(bucket_capacity=CAP))
    return import_state(gi, data["X"], data["S"], gold["adj"], gold["boundaries"], i2b, lists, N)


@pytest.fixture(scope="module")
def gref(g, data, gold):
    return ref_graph(g, data, gold)


def _recall(g, gi, Q, lo, hi, params):
    from paper_2604_16402_b200.datasets import batch_recall
    r = g.search_arrays(gi, Q, lo, hi, params, seed_base=3, stats=False)
    ts, _, tc = g.brute_force_arrays(gi, Q, lo, hi, params.k)
    return batch_recall(r.slots, r.counts, ts, tc, params.k)


def test_cfg1_partition_matches_reference(g, data, gold):
    meta = g.partition_buckets(data["S"], CAP)
    assert meta.m == 16
    assert meta.boundaries.tobytes() == gold["boundaries"].tobytes()
    assert np.array_equal(meta.index_to_bucket[:N], gold["i2b"].astype(np.int32))


def test_cfg1_search_matches_reference_all_modes(g, data, gold, gref):
    import torch
    Q = data["Q"]
    for si in range(len(SELS)):
        lo, hi = gold[f"sel{si}_lower"], gold[f"sel{si}_upper"]
        for gidx, p in enumerate(GRID):
            params = g.SearchParams(**p)
            key = f"sel{si}_g{gidx}_"
            res = g.search_arrays(gref, Q, lo, hi, params, seed_base=11)
            assert np.array_equal(res.counts.astype(np.int32), gold[key + "counts"]), (si, gidx)
            for i in range(len(Q)):
                c = int(res.counts[i])
                assert np.array_equal(res.slots[i, :c], gold[key + "slots"][i, :c]), (si, gidx, i)
                np.testing.assert_allclose(res.dists[i, :c], gold[key + "dists"][i, :c], rtol=1e-12, atol=0)
                assert [int(res.stats[i][f]) for f in STAT_KEYS] == gold[key + "stats"][i].tolist(), (si, gidx, i)
            assert np.array_equal((res.counts > 0) & (res.counts < p["k"]), gold[key + "truncated"])
            # the stats-free kernel instance (insert candidate search, stats=False callers)
            r0 = g.search_arrays(gref, Q, lo, hi, params, seed_base=11, stats=False)
            assert np.array_equal(r0.slots, res.slots) and np.array_equal(r0.dists, res.dists, equal_nan=True)
            # page-locked host buffers (zero-copy kernel path) and device-resident buffers
            Qp = torch.from_numpy(Q).pin_memory()
            rp = g.search_arrays(gref, Qp, lo, hi, params, seed_base=11)
            assert np.array_equal(np.asarray(rp.slots), res.slots)
            Qd = torch.from_numpy(Q).cuda()
            rd = g.search_arrays(gref, Qd, torch.from_numpy(lo).cuda(), torch.from_numpy(hi).cuda(), params,
                                 seed_base=11)
            torch.cuda.synchronize()
            assert np.array_equal(rd.slots.cpu().numpy(), res.slots)
            assert np.array_equal(rd.dists.cpu().numpy(), res.dists, equal_nan=True)


def test_cfg1_bruteforce_matches_reference(g, data, gold, gref):
    for si in range(len(SELS)):
        lo, hi = gold[f"sel{si}_lower"], gold[f"sel{si}_upper"]
        s, _, c = g.brute_force_arrays(gref, data["Q"], lo, hi, 10)
        want = gold[f"sel{si}_bf_slots"]
        for i in range(len(data["Q"])):
            assert np.array_equal(s[i, : int(c[i])], want[i][want[i] >= 0]), (si, i)


def test_cfg1_workload_slots_and_recall(g, data, gold, gref):
    """configs[0] itself: 1K queries at 10 %, default SearchParams, search_batch seeds."""
    from paper_2604_16402_b200.datasets import batch_recall, generate_ranges, range_arrays
    lo, hi = range_arrays(generate_ranges(data["S"], 0.1, 1000, 0))
    params = g.SearchParams()
    r = g.search_arrays(gref, data["Q1"], lo, hi, params, seed_base=0)
    assert np.array_equal(r.counts.astype(np.int32), gold["w_counts"])
    assert np.array_equal(r.slots, gold["w_slots"])
    ts, _, tc = g.brute_force_arrays(gref, data["Q1"], lo, hi, 10)
    assert batch_recall(r.slots, r.counts, ts, tc, 10) == pytest.approx(float(gold["w_recall"]), abs=1e-12)


def test_cfg1_gpu_build_recall_within_tolerance(g, data, gold, gref):
    from paper_2604_16402_b200.datasets import generate_ranges, range_arrays
    gb, rep = g.build_index(data["X"], data["S"], g.BuildParams(bucket_capacity=CAP))
    assert rep.m == 16 and rep.global_pass == "exact"  # n <= 100 000: the reference's exact global pass
    same = np.mean(np.all(gb.adjacency[:N] == gold["adj"], axis=1))
    print(f"cfg1 GPU-built rows identical to the reference-built graph: {same:.5f}")
    assert same >= 0.99
    for sel in SELS:
        lo, hi = range_arrays(generate_ranges(data["S"], sel, len(data["Qr"]), 0))
        for p in (g.SearchParams(), g.SearchParams(itopk=64, max_iterations=30)):
            r_ref = _recall(g, gref, data["Qr"], lo, hi, p)
            r_gpu = _recall(g, gb, data["Qr"], lo, hi, p)
            print(f"sel {sel} itopk {p.itopk}: recall reference-built {r_ref:.4f} GPU-built {r_gpu:.4f}")
            assert abs(r_gpu - r_ref) <= RECALL_TOL, (sel, p.itopk, r_ref, r_gpu)


def test_cfg1_insert_matches_reference(g, data, golden):
    """20K rows inserted as the reference's four 5K batches (as many as the
    golden holds): every InsertReport, rewired-row set, and adjacency row."""
    gold = golden("cfg1_insert")
    nb = int(gold["ins_batches"])
    per = N_INS // INS_BATCHES
    gi = ref_graph(g, data, golden("cfg1"))
    for b in range(nb):
        rep = g.insert_batch(gi, data["Vn"][b * per:(b + 1) * per], data["Sn"][b * per:(b + 1) * per])
        assert [getattr(rep, k) for k in INSERT_KEYS] == gold[f"ins{b}_report"].tolist(), b
        assert np.array_equal(np.array(sorted(rep.rewired_rows), np.uint32), gold[f"ins{b}_rewired"]), b
    h = row_hash(gi.adjacency[: N + nb * per])
    same = float(np.mean(h == gold["ins_row_hash"]))
    print(f"cfg1 insert ({nb} x {per}): rows identical to the reference's {same:.6f}")
    assert same == 1.0


def test_cfg1_gpu_build_and_insert_recall_within_tolerance(g, data, gold):
    from paper_2604_16402_b200.datasets import generate_ranges, range_arrays
    per = N_INS // INS_BATCHES
    gi_ref = ref_graph(g, data, gold)
    gb, _ = g.build_index(data["X"], data["S"], g.BuildParams(bucket_capacity=CAP))
    for b in range(INS_BATCHES):  # on gi_ref: the reference's inserts (previous test, row for row)
        for gi in (gi_ref, gb):
            g.insert_batch(gi, data["Vn"][b * per:(b + 1) * per], data["Sn"][b * per:(b + 1) * per])
    S_all = np.concatenate([data["S"], data["Sn"]])
    for sel in SELS:
        lo, hi = range_arrays(generate_ranges(S_all, sel, len(data["Qr"]), 0))
        p = g.SearchParams()
        r_ref = _recall(g, gi_ref, data["Qr"], lo, hi, p)
        r_gpu = _recall(g, gb, data["Qr"], lo, hi, p)
        print(f"sel {sel}: recall after insert, reference {r_ref:.4f} GPU {r_gpu:.4f}")
        assert abs(r_gpu - r_ref) <= RECALL_TOL, (sel, r_ref, r_gpu)
