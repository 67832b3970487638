"""GPU build parity: device build_index vs the reference (goldens) and the
oracle restatement (oracle/construct.py) on identical inputs."""
import numpy as np
import pytest

from oracle import beam, construct, index_state as ist

pytestmark = pytest.mark.gpu
SENT = 0xFFFFFFFF


@pytest.fixture(scope="module")
def g():
    import paper_2604_16402_b200 as g
    return g


def f64_knn(X, k):
    X = X.astype(np.float64)
    d = ((X[:, None, :] - X[None, :, :]) ** 2).sum(-1)
    np.fill_diagonal(d, np.inf)
    n = len(X)
    return np.array([np.lexsort((np.arange(n), d[i]))[: min(k, n - 1)] for i in range(n)]), d


def test_pass1_forward_rows_equal_f64_oracle(g):
    r = np.random.default_rng(7)
    V = r.standard_normal((200, 8)).astype(np.float32)
    S = r.random(200, dtype=np.float32)
    gi, rep, dr = g.build_index(V, S, g.BuildParams(k_max=32, k_local=16, bucket_capacity=200), return_draft=True)
    want, _ = f64_knn(V, 32)
    assert rep.m == 1
    assert np.array_equal(dr.forward_rows.astype(np.int64), want)


def test_pass1_three_collinear_points(g):
    V = np.array([[0.0], [1.0], [3.0]], np.float32)
    gi, _, dr = g.build_index(V, np.array([0.1, 0.2, 0.3], np.float32),
                              g.BuildParams(k_max=2, k_local=1, bucket_capacity=10), return_draft=True)
    assert dr.forward_rows.tolist() == [[1, 2], [0, 2], [1, 0]]


def test_pass1_merged_rows_follow_interleave_rule(g):
    r = np.random.default_rng(8)
    V = r.standard_normal((40, 4)).astype(np.float32)
    S = r.random(40, dtype=np.float32)
    gi, _, dr = g.build_index(V, S, g.BuildParams(k_max=8, k_local=4, bucket_capacity=40), return_draft=True)
    fwd, d = f64_knn(V, 8)
    rev = {u: [] for u in range(40)}
    for u in range(40):
        for v in fwd[u]:
            rev[int(v)].append((d[v, u], u))
    for u in range(40):
        want = construct.interleave([int(x) for x in fwd[u]], [s for _, s in sorted(rev[u])], 8)
        assert [int(x) for x in dr.rows[u] if x != SENT] == want
        assert dr.necessary_counts[u] == min(len(want), 4)


def test_singleton_bucket_is_isolated(g):
    V = np.array([[0.0], [1.0], [1.1]], np.float32)
    S = np.array([0.05, 0.8, 0.9], np.float32)
    gi, rep, dr = g.build_index(V, S, g.BuildParams(k_max=2, k_local=1, bucket_capacity=2), bucket_strategy="width",
                                return_draft=True)
    assert rep.m == 2 and rep.isolated_nodes == 1
    assert np.all(dr.rows[0] == SENT)


def test_global_graph_three_points_complete(g):
    V = np.array([[0.0, 0], [1, 0], [0, 1]], np.float32)
    gi, _, dr = g.build_index(V, np.array([0.1, 0.5, 0.9], np.float32),
                              g.BuildParams(k_max=2, k_local=1, bucket_capacity=10), k_g=2, return_draft=True)
    assert {tuple(sorted(int(x) for x in row)) for row in dr.global_rows} == {(1, 2), (0, 2), (0, 1)}


def _invariants(gi, k_local):
    n = gi.count
    A = gi.adjacency[:n]
    i2b = gi.meta.index_to_bucket
    for u in range(n):
        live = A[u][A[u] != SENT].astype(np.int64)
        assert u not in live
        assert len(set(live.tolist())) == len(live)
        for pos in range(k_local):
            if A[u, pos] != SENT:
                assert i2b[A[u, pos]] == i2b[u]
    flat = A[A != SENT].astype(np.int64)
    assert (np.bincount(flat, minlength=n) == 0).sum() == 0


def test_small_build_matches_reference(g, golden):
    gold = golden("small")
    ref = ist.index_from_container(gold["container"].tobytes())
    V, S = ist.gen_synthetic(2000, 8, "clusters", rng_seed=1)
    gi, rep, dr = g.build_index(V, S, g.BuildParams(k_max=16, k_local=8, bucket_capacity=250), return_draft=True)
    meta = gi.meta
    assert meta.boundaries.tobytes() == ref.boundaries.tobytes()
    assert np.array_equal(meta.index_to_bucket[:2000], ref.i2b[:2000])
    assert rep.bucket_sizes == [len(b) for b in ref.b2i]
    same_fwd = np.mean([np.array_equal(a, b) for a, b in zip(dr.forward_rows, gold["draft_forward"])])
    same_adj = np.mean([np.array_equal(a, b) for a, b in zip(gi.adjacency[:2000], ref.adjacency[:2000])])
    print(f"forward-row identity {same_fwd:.4f}  final-row identity {same_adj:.4f}")
    assert same_fwd == 1.0
    assert same_adj == 1.0
    _invariants(gi, 8)


def test_build_recall_parity_with_reference(g):
    """North-star bar: GPU-built index recall@10 within 0.005 of the reference-built one."""
    X, S = ist.gen_lowrank(20_000, 32, seed=0)
    Q = ist.lowrank_queries(400, 32, seed=1)
    cfg = ist.BuildCfg(k_max=32, k_local=16, bucket_capacity=2000)
    ref, _, _ = construct.build(X, S, cfg)
    params = g.BuildParams(k_max=32, k_local=16, bucket_capacity=2000)
    ref_gpu = g.load_index(ist.container_bytes(ref), params)
    gi, rep = g.build_index(X, S, params)
    _invariants(gi, 16)
    for sel in (0.1, 0.5):
        ranges = beam.window_ranges(S, sel, len(Q), 0)
        lo = np.array([r[0] for r in ranges])
        hi = np.array([r[1] for r in ranges])
        truth, _, tc = g.brute_force_arrays(gi, Q, lo, hi, 10)
        sp = g.SearchParams(k=10, itopk=64)
        a = g.search_arrays(gi, Q, lo, hi, sp, seed_base=0)
        b = g.search_arrays(ref_gpu, Q, lo, hi, sp, seed_base=0)
        ra = np.mean([beam.recall(a.slots[i, :a.counts[i]], truth[i, :tc[i]], 10) for i in range(len(Q))])
        rb = np.mean([beam.recall(b.slots[i, :b.counts[i]], truth[i, :tc[i]], 10) for i in range(len(Q))])
        print(f"sel {sel}: recall gpu-built {ra:.4f} reference-built {rb:.4f}")
        assert abs(ra - rb) <= 0.005


@pytest.mark.parametrize("kg,rounds,key", [(8, 0, "rows0"), (32, 3, "rows")])
def test_nn_descent_global_pass_matches_reference(g, golden, kg, rounds, key):
    """build_global_graph above the exact limit (builder.py:379-393): random init from
    default_rng([seed, 1]) regenerated on the device, numpy-shuffle hop columns,
    descent rounds and the reverse merge -- every global row identical to the
    reference's (golden from the live reference, exact_limit=0)."""
    want = golden("descent")[key]
    r = np.random.default_rng(9)
    V = r.standard_normal((2000, 16)).astype(np.float32)
    S = r.random(2000, dtype=np.float32)
    _, rep, dr = g.build_index(V, S, g.BuildParams(), k_g=kg, refine_rounds=rounds, return_draft=True,
                               global_pass="descent")
    assert rep.global_pass == "descent"
    assert np.array_equal(dr.global_rows, want)


def test_auto_global_pass_follows_reference_limit(g):
    r = np.random.default_rng(1)
    V = r.standard_normal((3000, 8)).astype(np.float32)
    S = r.random(3000, dtype=np.float32)
    _, rep = g.build_index(V, S, g.BuildParams(bucket_capacity=1000))
    assert rep.global_pass == "exact"  # n <= EXACT_GLOBAL_LIMIT (builder.py:33)
    _, rep = g.build_index(V, S, g.BuildParams(bucket_capacity=1000), global_pass="descent")
    assert rep.global_pass == "descent"


def test_partition_buckets_matches_reference_goldens(g, golden):
    """partition_buckets (layout.py:107-154) on the device: boundaries byte-identical
    and M_I2B / M_B2I equal to the live reference's on every golden case
    (quantile, skewed, all-equal, width, ties, odd n)."""
    gl = golden("layout")
    cases = {
        "uniform": (np.random.default_rng(0).random(10_000, dtype=np.float32), 1000, "quantile"),
        "skewed": ((np.random.default_rng(3).random(5000, dtype=np.float32) ** 8).astype(np.float32), 500, "quantile"),
        "equal": (np.full(100, 5.0, np.float32), 10, "quantile"),
        "width": (np.random.default_rng(2).random(1000, dtype=np.float32), 100, "width"),
        "ties": (np.round(np.random.default_rng(4).random(3000) * 20).astype(np.float32), 97, "quantile"),
        "odd": (np.random.default_rng(5).standard_normal(1237).astype(np.float32), 100, "quantile"),
    }
    for name, (s, cap, strat) in cases.items():
        meta = g.partition_buckets(s, cap, strategy=strat, capacity=len(s) + 7)
        assert meta.boundaries.tobytes() == gl[f"{name}_boundaries"].tobytes(), name
        assert np.array_equal(meta.index_to_bucket[: len(s)], gl[f"{name}_i2b"][: len(s)]), name
        assert (meta.index_to_bucket[len(s):] == -1).all()
        flat = [slot for b in meta.bucket_to_index for slot in b]
        assert sorted(flat) == list(range(len(s))) and all(b == sorted(b) for b in meta.bucket_to_index)
        assert all(meta.index_to_bucket[x] == bi for bi, b in enumerate(meta.bucket_to_index) for x in b)
    with pytest.raises(ValueError):
        g.partition_buckets(np.zeros(0, np.float32), 10)


@pytest.mark.parametrize("n,d,kg,rounds", [(30_000, 32, 32, 3), (12_000, 200, 16, 2), (5_000, 8, 8, 1)])
def test_split_descent_rounds_equal_direct_rounds(g, n, d, kg, rounds):
    """descent.cu's split round (per-hop-source f32 screen, exact rerank of the
    columns that can still be in the top k) returns the direct round's rows
    bit for bit: same global rows, same final adjacency."""
    import os
    from paper_2604_16402_b200.datasets import gen_lowrank
    X, S = gen_lowrank(n, d, seed=11)
    params = g.BuildParams(k_max=32, k_local=16, bucket_capacity=max(1000, n // 10))
    out = {}
    for mode in ("direct", "split"):
        if mode == "direct":
            os.environ["GRAB_DESCENT_DIRECT"] = "1"
        try:
            gi, rep, dr = g.build_index(X, S, params, k_g=kg, refine_rounds=rounds, return_draft=True,
                                        global_pass="descent")
        finally:
            os.environ.pop("GRAB_DESCENT_DIRECT", None)
        out[mode] = (dr.global_rows.copy(), gi.adjacency[:n].copy())
    assert np.array_equal(out["split"][0], out["direct"][0])
    assert np.array_equal(out["split"][1], out["direct"][1])
