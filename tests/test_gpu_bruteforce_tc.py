"""Tensor-core brute force (bruteforce.cu run_bruteforce -> knn_tc.cu BF screen +
f64 rerank + completeness proof) against the SIMT scan (GRAB_BF_SIMT=1), which
the goldens pin to the reference's brute_force_search (evaluate.py:22-44).

The bar is bit-exact: identical slots, counts and f64 distances for every
query -- wide / narrow / empty / inverted / shared ranges, short results
(fewer than k rows in range), k = 1 .. 64, d = 8 / 128 / 960, a live_count
below the published count, and an index with inserted rows (slab headroom in
the span)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _both(g, gi, Q, lo, hi, k, live=None):
    os.environ["GRAB_BF_SIMT"] = "1"
    os.environ.pop("GRAB_BF_DEBUG", None)
    try:
        ref = g.brute_force_arrays(gi, Q, lo, hi, k, live_count=live)
    finally:
        del os.environ["GRAB_BF_SIMT"]
    os.environ["GRAB_BF_DEBUG"] = "1"
    try:
        got = g.brute_force_arrays(gi, Q, lo, hi, k, live_count=live)
    finally:
        del os.environ["GRAB_BF_DEBUG"]
    return ref, got


def _reruns(capfd):
    """SIMT re-runs reported by the tensor-core path since the last call (GRAB_BF_DEBUG)."""
    err = capfd.readouterr().err
    lines = [ln for ln in err.splitlines() if "brute force tc:" in ln]
    assert lines, "the tensor-core path did not run"
    return [int(ln.rsplit(" ", 1)[1]) for ln in lines]


def _assert_same(ref, got):
    rs, rd, rc = ref
    gs, gd, gc = got
    assert np.array_equal(rc, gc)
    assert np.array_equal(rs, gs)
    assert np.array_equal(rd, gd, equal_nan=True)


@pytest.fixture(scope="module")
def g():
    import paper_2604_16402_b200 as g
    return g


@pytest.mark.parametrize("dim,n,cap", [(128, 60_000, 2_000), (8, 20_000, 1_000), (960, 12_000, 1_500)])
def test_tc_bruteforce_equals_simt(g, dim, n, cap, capfd):
    from paper_2604_16402_b200 import datasets as ds
    X, S = ds.gen_lowrank(n, dim, seed=3)
    gi, _ = g.build_index(X, S, g.BuildParams(k_max=16, k_local=8, bucket_capacity=cap))
    nq = 700
    Q = ds.lowrank_queries(nq, dim, seed=4)
    rng = np.random.default_rng(5)
    for sel in (0.5, 0.1, 0.01, 0.0005):
        lo = rng.random(nq) * (1 - sel)
        hi = lo + sel
        lo[::97] = 0.7   # inverted / empty ranges mixed in
        hi[::97] = 0.2
        lo[1::89] = 2.0  # above every scalar
        hi[1::89] = 3.0
        for k in (1, 10, 64):
            ref, got = _both(g, gi, Q, lo, hi, k)
            _assert_same(ref, got)
            rr = _reruns(capfd)
            print(f"d {dim} sel {sel} k {k}: simt re-runs {rr}")
            assert rr[0] <= nq // 20  # the proof holds for (nearly) every query
    # one shared range for the batch (range_stride 0)
    ref, got = _both(g, gi, Q, np.array([0.25]), np.array([0.4]), 10)
    _assert_same(ref, got)


def test_tc_bruteforce_after_insert_and_live_count(g, capfd):
    from paper_2604_16402_b200 import datasets as ds
    X, S = ds.gen_lowrank(30_000, 64, seed=6)
    gi, _ = g.build_index(X[:20_000], S[:20_000], g.BuildParams(k_max=16, k_local=8, bucket_capacity=2_000))
    g.insert_batch(gi, X[20_000:], S[20_000:])
    Q = ds.lowrank_queries(300, 64, seed=7)
    rng = np.random.default_rng(8)
    lo = rng.random(300) * 0.8
    hi = lo + 0.2
    for live in (None, 25_000, 5):
        ref, got = _both(g, gi, Q, lo, hi, 10, live)
        _assert_same(ref, got)
        assert _reruns(capfd)[0] <= 15
