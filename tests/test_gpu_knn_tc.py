"""tcgen05 kNN screen vs the SIMT screen and the f64 oracle (same build outputs)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import index_state as ist

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def f64_knn(X, k):
    X = X.astype(np.float64)
    d = ((X[:, None, :] - X[None, :, :]) ** 2).sum(-1)
    np.fill_diagonal(d, np.inf)
    n = len(X)
    return np.array([np.lexsort((np.arange(n), d[i]))[: min(k, n - 1)] for i in range(n)])


@pytest.mark.parametrize("d", [8, 16, 96, 128, 200, 384, 960])
def test_tc_pass1_equals_f64_oracle(d):
    """d > 128 streams A through the ring one K chunk at a time (TMEM accumulates)."""
    import paper_2604_16402_b200 as g
    r = np.random.default_rng(7 + d)
    V = r.standard_normal((700, d)).astype(np.float32)
    S = r.random(700, dtype=np.float32)
    gi, rep, dr = g.build_index(V, S, g.BuildParams(k_max=32, k_local=16, bucket_capacity=700), return_draft=True)
    want = f64_knn(V, 32)
    assert np.array_equal(dr.forward_rows.astype(np.int64), want)
    assert np.array_equal(dr.global_rows[:, :1].astype(np.int64), want[:, :1])


def _build_draft(env_simt: bool, seed: int, dim: int = 128):
    code = f"""
import sys, numpy as np
sys.path.insert(0, {ROOT!r})
import paper_2604_16402_b200 as g
from oracle import index_state as ist
X, S = ist.gen_lowrank(30000, {dim}, seed={seed})
gi, rep, dr = g.build_index(X, S, g.BuildParams(k_max=32, k_local=16, bucket_capacity=3000), return_draft=True)
np.savez(sys.argv[1], f=dr.forward_rows, m=dr.rows, g=dr.global_rows, a=gi.adjacency[:gi.count])
"""
    out = f"/tmp/draft_{int(env_simt)}_{seed}_{dim}.npz"
    env = dict(os.environ)
    if env_simt:
        env["GRAB_KNN_SIMT"] = "1"
    else:
        env.pop("GRAB_KNN_SIMT", None)
    subprocess.run([sys.executable, "-c", code, out], check=True, env=env)
    return np.load(out)


@pytest.mark.parametrize("dim", [128, 960])
def test_tc_build_matches_simt_build(dim):
    a = _build_draft(False, 5, dim)
    b = _build_draft(True, 5, dim)
    for key in ("f", "g", "m", "a"):
        same = np.mean([np.array_equal(x, y) for x, y in zip(a[key], b[key])])
        print(key, same)
        assert same >= 0.999, key
