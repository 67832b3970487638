"""Harness / formats / CLI (reference evaluate.py, dataio.py:1-108, cli.py):
CPU checks of the host formats and argument surface; GPU checks of the device
SCC count (vs scipy's strong components), the batched sweep and the CLI."""
import json
import os
import struct
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT


def test_fvecs_and_scalars_round_trip(tmp_path):
    from paper_2604_16402_b200 import dataio
    v = np.random.default_rng(0).standard_normal((7, 5)).astype(np.float32)
    p = tmp_path / "a.fvecs"
    dataio.write_fvecs(p, v)
    assert p.stat().st_size == 7 * (4 + 4 * 5)
    assert np.array_equal(dataio.read_fvecs(p), v)
    s = np.arange(9, dtype=np.float32) / 3
    dataio.write_scalars(tmp_path / "s.f32", s)
    assert np.array_equal(dataio.read_scalars(tmp_path / "s.f32"), s)


def test_fvecs_errors_report_byte_offsets(tmp_path):
    from paper_2604_16402_b200 import dataio
    p = tmp_path / "bad.fvecs"
    rec = struct.pack("<i", 2) + struct.pack("<ff", 1, 2)
    p.write_bytes(rec + struct.pack("<i", 3) + struct.pack("<ff", 1, 2))
    with pytest.raises(dataio.FvecsFormatError) as e:
        dataio.read_fvecs(p)
    assert e.value.offset == 12
    p.write_bytes(rec + b"\x00\x00")
    with pytest.raises(dataio.FvecsFormatError) as e:
        dataio.read_fvecs(p)
    assert e.value.offset == 12
    (tmp_path / "s").write_bytes(struct.pack("<Q", 3) + b"\x00" * 8)
    with pytest.raises(ValueError):
        dataio.read_scalars(tmp_path / "s")


def test_gt_cache_file_format(tmp_path):
    from paper_2604_16402_b200.evaluate import GroundTruthCache
    c = GroundTruthCache(tmp_path)
    truth = [np.array([3, 1, 2]), np.array([], dtype=np.int64), np.array([9])]
    c._write(tmp_path / "x.gt", truth, 10)
    raw = (tmp_path / "x.gt").read_bytes()
    assert raw[:4] == b"GTC1" and struct.unpack_from("<II", raw, 4) == (3, 10)
    back = c._read(tmp_path / "x.gt")
    assert [b.tolist() for b in back] == [t.tolist() for t in truth]


def test_cli_parser_mirrors_reference():
    from paper_2604_16402_b200 import cli
    p = cli._build_parser()
    a = p.parse_args(["build", "--data", "d", "--scalars", "s", "--out", "o"])
    assert (a.kmax, a.klocal, a.bucket_cap, a.alpha, a.headroom, a.bucket_strategy) == (32, 16, 10000, 0.6, 2.0,
                                                                                         "quantile")
    a = p.parse_args(["query", "--index", "i", "--queries", "q"])
    assert (a.k, a.itopk, a.width, a.max_iter) == (10, 128, 4, 50)
    r = subprocess.run([sys.executable, "-m", "paper_2604_16402_b200.cli", "nope"], capture_output=True, text=True,
                       cwd=ROOT)
    assert r.returncode == 2 and json.loads(r.stderr.strip())["error"] == "usage"


@pytest.mark.gpu
def test_scc_count_matches_strong_components():
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components

    import paper_2604_16402_b200 as g
    from paper_2604_16402_b200 import datasets as ds
    from paper_2604_16402_b200.evaluate import scc_count
    for dist, n in (("clusters", 4000), ("gaussian", 3000)):
        V, S = ds.gen_synthetic(n, 16, dist, rng_seed=3)
        gi, _ = g.build_index(V, S, g.BuildParams(k_max=16, k_local=8, bucket_capacity=400))
        A = gi.adjacency[:n]
        ok = A != 0xFFFFFFFF
        rows = np.repeat(np.arange(n), A.shape[1])[ok.ravel()]
        cols = A.ravel()[ok.ravel()].astype(np.int64)
        m = csr_matrix((np.ones(len(rows)), (rows, cols)), shape=(n, n))
        want = connected_components(m, directed=True, connection="strong")[0]
        assert scc_count(gi) == want
        assert scc_count(A, n) == want
    # hand graph: 0<->1, 2 -> 0, 3 alone, edges past live_count ignored
    A = np.full((5, 2), 0xFFFFFFFF, dtype=np.uint32)
    A[0, 0], A[1, 0], A[2, 0], A[3, 0] = 1, 0, 0, 4
    assert scc_count(A, 4) == 3


@pytest.mark.gpu
def test_run_sweep_and_cli_end_to_end(tmp_path):
    import paper_2604_16402_b200 as g
    from paper_2604_16402_b200 import datasets as ds, evaluate
    X, S = ds.gen_lowrank(6000, 32, seed=0)
    gi, _ = g.build_index(X, S, g.BuildParams(k_max=16, k_local=8, bucket_capacity=600))
    Q = ds.lowrank_queries(64, 32, seed=1)
    spec = evaluate.SweepSpec(selectivities=[0.1, 1.0], itopk_values=[32, 128], query_count=64)
    cache = evaluate.GroundTruthCache(tmp_path / "gt")
    rep = evaluate.run_sweep(gi, Q, spec, gt_cache=cache)
    assert len(rep.rows) == 4 and len(list((tmp_path / "gt").glob("*.gt"))) == 2
    by = {(r["selectivity"], r["itopk"]): r["recall"] for r in rep.rows}
    assert by[(0.1, 128)] >= by[(0.1, 32)] - 0.005 and by[(0.1, 128)] > 0.9
    rep.write_csv(tmp_path / "s.csv")
    assert (tmp_path / "s.csv").read_text().splitlines()[0].split(",")[0] == "selectivity"
    # CLI: gen -> build -> query -> insert -> analyze
    env = dict(os.environ, PYTHONPATH=ROOT)
    run = lambda *a: subprocess.run([sys.executable, "-m", "paper_2604_16402_b200.cli", *a], capture_output=True,
                                    text=True, cwd=ROOT, env=env, timeout=300)
    pre = str(tmp_path / "ds")
    r = run("gen", "--n", "3000", "--d", "16", "--n-queries", "5", "--out", pre)
    assert r.returncode == 0, r.stderr
    r = run("build", "--data", pre + ".base.fvecs", "--scalars", pre + ".scalars.f32", "--bucket-cap", "500",
            "--out", str(tmp_path / "i.grab"))
    assert r.returncode == 0 and json.loads(r.stdout)["indexed"] == 3000, r.stderr
    r = run("query", "--index", str(tmp_path / "i.grab"), "--queries", pre + ".queries.fvecs", "--range", "0.2,0.6")
    lines = [json.loads(x) for x in r.stdout.splitlines()]
    assert r.returncode == 0 and len(lines) == 5 and len(lines[0]["slots"]) == 10
    r = run("insert", "--index", str(tmp_path / "i.grab"), "--data", pre + ".queries.fvecs", "--scalars",
            pre + ".scalars.f32")
    assert r.returncode == 1 and json.loads(r.stderr)["error"] == "ValueError"  # 5 vectors vs 3000 scalars
    r = run("analyze", "--index", str(tmp_path / "i.grab"))
    assert r.returncode == 0 and json.loads(r.stdout)["count"] == 3000
    r = run("analyze", "--index", str(tmp_path / "i.grab"), "--scc")
    assert r.returncode == 0 and int(r.stdout) >= 1
