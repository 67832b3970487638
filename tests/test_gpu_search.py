"""GPU parity: search / brute force / bucket selection through the C ABI versus
golden vectors frozen from the live reference (tests/golden/make_golden.py)."""
import numpy as np
import pytest

from oracle import beam, index_state as ist

pytestmark = pytest.mark.gpu

GRID = [dict(k=10, itopk=128, search_width=4, max_iterations=50),
        dict(k=10, itopk=32, search_width=1, max_iterations=50),
        dict(k=5, itopk=64, search_width=2, max_iterations=10),
        dict(k=16, itopk=256, search_width=4, max_iterations=100)]
STAT_KEYS = ["iterations", "dist_evals", "seed_evals", "gathered", "in_range_new", "precheck_rejected",
             "seed_attempts"]


@pytest.fixture(scope="module")
def g():
    import paper_2604_16402_b200 as g
    return g


def _compare_grid(g, gi, Q, prefix, gold):
    for si in range(4):
        lo, hi = gold[f"{prefix}_sel{si}_lower"], gold[f"{prefix}_sel{si}_upper"]
        for gidx, p in enumerate(GRID):
            params = g.SearchParams(**p)
            res = g.search_arrays(gi, Q, lo, hi, params, seed_base=11)
            key = f"{prefix}_sel{si}_g{gidx}_"
            assert np.array_equal(res.counts.astype(np.int32), gold[key + "counts"]), (si, gidx)
            for i in range(len(Q)):
                c = int(res.counts[i])
                assert np.array_equal(res.slots[i, :c], gold[key + "slots"][i, :c]), (si, gidx, i)
                np.testing.assert_allclose(res.dists[i, :c], gold[key + "dists"][i, :c], rtol=1e-12, atol=0)
                got = [int(res.stats[i][f]) for f in STAT_KEYS]
                assert got == gold[key + "stats"][i].tolist(), (si, gidx, i)
            tr = (res.counts > 0) & (res.counts < p["k"])
            assert np.array_equal(tr, gold[key + "truncated"])
        s, d, c = g.brute_force_arrays(gi, Q, lo, hi, 10)
        want_s = gold[f"{prefix}_sel{si}_bf_slots"]
        for i in range(len(Q)):
            n = int(c[i])
            assert np.array_equal(s[i, :n], want_s[i][want_s[i] >= 0])
            np.testing.assert_allclose(d[i, :n], gold[f"{prefix}_sel{si}_bf_dists"][i, :n], rtol=1e-12, atol=0)


def test_small_index_search_matches_reference(g, golden):
    gold = golden("small")
    gi = g.load_index(gold["container"].tobytes(), g.BuildParams(k_max=16, k_local=8, bucket_capacity=250))
    Q, _ = ist.gen_synthetic(64, 8, "clusters", rng_seed=1)
    _compare_grid(g, gi, Q + np.float32(0.01), "s", gold)


def test_mid_index_search_matches_reference(g, golden):
    gold = golden("mid")
    gi = g.load_index(gold["container"].tobytes())
    V, _ = ist.gen_synthetic(10_120, 16, "clusters", rng_seed=2)
    _compare_grid(g, gi, V[10_000:10_048], "m", gold)


def test_batch_shared_range_and_edges(g, golden):
    gold = golden("small")
    gi = g.load_index(gold["container"].tobytes(), g.BuildParams(k_max=16, k_local=8, bucket_capacity=250))
    Q, _ = ist.gen_synthetic(64, 8, "clusters", rng_seed=1)
    Q = Q + np.float32(0.01)
    res = g.search_batch(gi, Q, g.SearchParams(k=10, range=g.RangePredicate(0.2, 0.45), itopk=64, rng_seed=21))
    for i, r in enumerate(res):
        c = gold["s_batch_counts"][i]
        assert np.array_equal(r.slots, gold["s_batch_slots"][i, :c])
    V, S = ist.gen_synthetic(2000, 8, "clusters", rng_seed=1)
    srt = np.sort(S)
    edges = [(2.0, 3.0), (float(srt[0]), float(srt[2])), (-np.inf, np.inf), (float(srt[0]), float(srt[-1]))]
    for i, (lo, hi) in enumerate(edges):
        r = g.search(gi, V[0], g.SearchParams(k=10, range=g.RangePredicate(lo, hi), itopk=64, rng_seed=5))
        c = gold["edge_counts"][i]
        assert np.array_equal(r.slots, gold["edge_slots"][i, :c])
        assert r.truncated == bool(gold["edge_truncated"][i])


def test_distance_soundness_is_bitwise(g, golden):
    gold = golden("mid")
    gi = g.load_index(gold["container"].tobytes())
    V, S = ist.gen_synthetic(10_120, 16, "clusters", rng_seed=2)
    Q = V[10_000:10_060]
    ranges = beam.window_ranges(S[:10_000], 0.2, len(Q), 11)
    X = gi.store.X
    for i, (lo, hi) in enumerate(ranges):
        r = g.search(gi, Q[i], g.SearchParams(k=10, range=g.RangePredicate(lo, hi), rng_seed=i))
        s = gi.store.scalars[r.slots]
        assert np.all((s >= np.float32(lo)) & (s <= np.float32(hi)))
        for slot, d in zip(r.slots, r.sq_dists):
            assert d == g.sq_distance(Q[i], X[slot])
        assert r.stats.dist_evals == r.stats.seed_evals + r.stats.in_range_new


def test_container_roundtrip_and_views(g, golden, tmp_path):
    gold = golden("small")
    raw = gold["container"].tobytes()
    gi = g.load_index(raw, g.BuildParams(k_max=16, k_local=8, bucket_capacity=250))
    p = tmp_path / "x.grab"
    g.save_index(gi, p)
    assert p.read_bytes() == raw
    ref = ist.index_from_container(raw)
    assert [len(x) for x in gi.meta.bucket_to_index] == [len(x) for x in ref.b2i]
    assert gi.meta.bucket_to_index == ref.b2i


def test_bucket_selection_bit_exact(g, golden):
    gold = golden("layout")
    meta = g.BucketMeta(boundaries=gold["iv_boundaries"], index_to_bucket=np.empty(0, np.int32),
                        bucket_to_index=[])
    for lo, hi, want in zip(gold["iv_lower"], gold["iv_upper"], gold["iv_lohi"]):
        assert g.intersecting_buckets(meta, g.RangePredicate(float(lo), float(hi))) == tuple(want)
    assert np.array_equal(g.bucket_ids_of(meta, gold["bid_scalars"]), gold["bid_ids"])


def test_search_empty_index(g):
    gi = g.create_index(4, 16, g.BuildParams(k_max=4, k_local=2))
    r = g.search(gi, np.zeros(4, np.float32), g.SearchParams(k=3, itopk=8))
    assert len(r) == 0 and not r.truncated


def _oracle_of(gi):
    p = gi.params
    n = gi.count
    meta = gi.meta
    return ist.OracleIndex(X=np.ascontiguousarray(gi.store.X[:n]), scalars=np.ascontiguousarray(gi.store.scalars[:n]),
                           ids=np.arange(n), count=n, adjacency=np.ascontiguousarray(gi.adjacency[:n]),
                           cfg=ist.BuildCfg(k_max=p.k_max, k_local=p.k_local, bucket_capacity=p.bucket_capacity),
                           boundaries=meta.boundaries, i2b=meta.index_to_bucket[:n], b2i=meta.bucket_to_index)


@pytest.mark.parametrize("mode", ["hash", "bitmap", "overflow"])
def test_wide_ranges_use_exact_hash_visited_set(g, mode, monkeypatch):
    """Ranges whose slab interval exceeds the warp's itopk-sized table (here >
    131K rows at itopk 64) use the open-addressing hash -- on indexes above 4M
    rows always, here forced with GRAB_SEARCH_HASH_VISITED -- or, when every phys
    row fits a bitmap, a full-span bitmap; results and every SearchStats counter
    must equal the oracle in both modes (searcher.py:156-233)."""
    if mode in ("hash", "overflow"):
        monkeypatch.setenv("GRAB_SEARCH_HASH_VISITED", "1")
    if mode == "overflow":  # a 512-entry table: wide queries pass 3/4 load and are re-run exactly
        monkeypatch.setenv("GRAB_SEARCH_VLOG2", "9")
    V, S = ist.gen_synthetic(300_000, 16, "gaussian", rng_seed=4)
    gi, _ = g.build_index(V, S, g.BuildParams(k_max=16, k_local=8, bucket_capacity=3000))
    ox = _oracle_of(gi)
    Q, _ = ist.gen_synthetic(12, 16, "gaussian", rng_seed=5)
    for lo, hi in ((-1.0, 2.0), (0.1, 0.8)):
        p = g.SearchParams(k=10, itopk=64, search_width=4, max_iterations=50)
        res = g.search_arrays(gi, Q, lo, hi, p, seed_base=3)
        fast = g.search_arrays(gi, Q, lo, hi, p, seed_base=3, stats=False)  # no per-iteration unique pass
        assert np.array_equal(fast.slots, res.slots) and np.array_equal(fast.dists, res.dists)
        for i in range(len(Q)):
            want = beam.beam_search(ox, Q[i], ist.SearchCfg(k=10, lower=lo, upper=hi, itopk=64, search_width=4,
                                                            max_iterations=50, rng_seed=beam.derive_seed(3, i)))
            c = int(res.counts[i])
            assert np.array_equal(res.slots[i, :c], want.slots), (lo, i)
            np.testing.assert_allclose(res.dists[i, :c], want.sq_dists, rtol=1e-12, atol=0)
            got = [int(res.stats[i][f]) for f in STAT_KEYS]
            ws = [getattr(want.stats, f) for f in STAT_KEYS]
            assert got == ws, (lo, i, got, ws)


def test_search_argument_errors_and_out_of_span(g, golden):
    gold = golden("small")
    gi = g.load_index(gold["container"].tobytes(), g.BuildParams(k_max=16, k_local=8, bucket_capacity=250))
    q = np.zeros(8, np.float32)
    with pytest.raises(ValueError):
        g.search_arrays(gi, q, 0.5, 0.4, g.SearchParams(k=10, itopk=64))  # lower > upper
    with pytest.raises(ValueError):
        g.search_arrays(gi, q, 0.0, 1.0, g.SearchParams(k=10, itopk=64, search_width=32))  # width*K > 256
    with pytest.raises(g.DimensionMismatchError):
        g.search_arrays(gi, np.zeros(9, np.float32), 0.0, 1.0, g.SearchParams(k=10, itopk=64))
    r = g.search_arrays(gi, np.stack([q, q]), np.array([5.0, -3.0]), np.array([6.0, -2.0]),
                        g.SearchParams(k=10, itopk=64))
    assert r.counts.tolist() == [0, 0] and (r.slots == -1).all()  # ranges outside the scalar span
    s, d, c = g.brute_force_arrays(gi, np.stack([q, q]), np.array([5.0, -3.0]), np.array([6.0, -2.0]), 10)
    assert c.tolist() == [0, 0]


def test_pinned_and_device_inputs_match_host(g, golden, monkeypatch):
    """Page-locked torch inputs (pinned results: zero-copy, and staged with
    GRAB_NO_ZERO_COPY=1) and device tensors give the host-array results bit for
    bit (the memory modes of grab_search)."""
    import torch
    gold = golden("mid")
    gi = g.load_index(gold["container"].tobytes())
    V, _ = ist.gen_synthetic(10_120, 16, "clusters", rng_seed=2)
    Q = np.ascontiguousarray(V[10_000:10_048])
    lo, hi = gold["m_sel1_lower"], gold["m_sel1_upper"]
    p = g.SearchParams(**GRID[0])
    ref = g.search_arrays(gi, Q, lo, hi, p, seed_base=11)
    pinned = (torch.from_numpy(Q).pin_memory(), torch.from_numpy(np.asarray(lo)).pin_memory(),
              torch.from_numpy(np.asarray(hi)).pin_memory())
    pin = g.search_arrays(gi, *pinned, p, seed_base=11)
    monkeypatch.setenv("GRAB_NO_ZERO_COPY", "1")
    staged = g.search_arrays(gi, *pinned, p, seed_base=11)
    monkeypatch.delenv("GRAB_NO_ZERO_COPY")
    dev = g.search_arrays(gi, torch.from_numpy(Q).cuda(), torch.from_numpy(np.asarray(lo)).cuda(),
                          torch.from_numpy(np.asarray(hi)).cuda(), p, seed_base=11)
    torch.cuda.synchronize()
    for r in (pin, staged, dev):
        sl = r.slots.cpu().numpy() if hasattr(r.slots, "cpu") else r.slots
        ds = r.dists.cpu().numpy() if hasattr(r.dists, "cpu") else r.dists
        ct = r.counts.cpu().numpy() if hasattr(r.counts, "cpu") else r.counts
        assert np.array_equal(ct.astype(np.int64), ref.counts.astype(np.int64))
        assert np.array_equal(sl, ref.slots) and np.array_equal(ds.view(np.int64), ref.dists.view(np.int64))
        if r.stats is not None and not hasattr(r.stats, "cpu"):
            assert r.stats.tobytes() == ref.stats.tobytes()


def test_concurrent_searches_match_sequential(g, golden):
    """Readers are concurrent-safe (SPEC: per-thread visited table): threads
    sharing the index -- host calls on the index stream, device calls on their
    own streams, with shapes that regrow the per-stream scratch -- return the
    sequential results."""
    import threading

    import torch
    gold = golden("mid")
    gi = g.load_index(gold["container"].tobytes())
    V, _ = ist.gen_synthetic(10_120, 16, "clusters", rng_seed=2)
    Q = np.ascontiguousarray(V[10_000:10_120])
    lo = np.concatenate([gold["m_sel2_lower"], gold["m_sel1_lower"], gold["m_sel3_lower"]])
    hi = np.concatenate([gold["m_sel2_upper"], gold["m_sel1_upper"], gold["m_sel3_upper"]])
    Qs = [Q[:48], Q[48:96], Q[72:120]]
    los = [lo[:48], lo[48:96], lo[72:120]]
    his = [hi[:48], hi[48:96], hi[72:120]]
    plist = [g.SearchParams(k=10, itopk=t, search_width=4, max_iterations=60) for t in (32, 128, 256, 512)]
    want = {(qi, pi): g.search_arrays(gi, Qs[qi], los[qi], his[qi], p, seed_base=7)
            for qi in range(3) for pi, p in enumerate(plist)}
    got, errs = {}, []

    def worker(tid):
        try:
            dev = tid % 2 == 1
            st = torch.cuda.Stream() if dev else None
            for rep in range(3):
                for qi in range(3):
                    for pi in ([0, 1, 2, 3] if (tid + rep) % 2 else [3, 2, 1, 0]):
                        if dev:
                            with torch.cuda.stream(st):
                                r = g.search_arrays(gi, torch.from_numpy(Qs[qi]).cuda(),
                                                    torch.from_numpy(np.asarray(los[qi])).cuda(),
                                                    torch.from_numpy(np.asarray(his[qi])).cuda(), plist[pi],
                                                    seed_base=7)
                                st.synchronize()
                            got[(tid, rep, qi, pi)] = r.slots.cpu().numpy()
                        else:
                            got[(tid, rep, qi, pi)] = g.search_arrays(gi, Qs[qi], los[qi], his[qi], plist[pi],
                                                                      seed_base=7).slots
        except Exception as e:  # pragma: no cover - reported below
            errs.append(repr(e))

    th = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    assert len(got) == 4 * 3 * 3 * 4
    for (tid, rep, qi, pi), sl in got.items():
        assert np.array_equal(sl, want[(qi, pi)].slots), (tid, rep, qi, pi)


@pytest.mark.parametrize("kmax,width", [(64, 4), (32, 8), (16, 16)])
def test_wide_fanout_search_matches_oracle(g, kmax, width):
    """search_width * K_max up to 256 (the paper's K_max = 64 with the default
    width 4): slots, f64 distances and every SearchStats counter equal the oracle."""
    V, S = ist.gen_synthetic(6_000, 16, "gaussian", rng_seed=8)
    gi, _ = g.build_index(V, S, g.BuildParams(k_max=kmax, k_local=kmax // 2, bucket_capacity=1000))
    ox = _oracle_of(gi)
    Q, _ = ist.gen_synthetic(16, 16, "gaussian", rng_seed=9)
    for lo, hi in ((-1.0, 2.0), (0.2, 0.5)):
        p = g.SearchParams(k=10, itopk=96, search_width=width, max_iterations=40)
        res = g.search_arrays(gi, Q, lo, hi, p, seed_base=5)
        for i in range(len(Q)):
            want = beam.beam_search(ox, Q[i], ist.SearchCfg(k=10, lower=lo, upper=hi, itopk=96, search_width=width,
                                                            max_iterations=40, rng_seed=beam.derive_seed(5, i)))
            c = int(res.counts[i])
            assert np.array_equal(res.slots[i, :c], want.slots), (kmax, width, lo, i)
            got = [int(res.stats[i][f]) for f in STAT_KEYS]
            assert got == [getattr(want.stats, f) for f in STAT_KEYS], (kmax, width, lo, i)
