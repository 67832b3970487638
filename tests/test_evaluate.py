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


SWEEP_SPEC = dict(selectivities=[0.01, 0.1, 0.5, 1.0], itopk_values=[32, 64], search_widths=[1, 4],
                  max_iterations_values=[10, 50], query_count=48, rng_seed=3)


def _sweep_inputs(golden):
    """small_index fixture + the sweep's queries (tests/golden/make_golden.py:sweep_golden)."""
    from oracle import index_state as ist
    gold = golden("small")
    ref = ist.index_from_container(gold["container"].tobytes())
    Q, _ = ist.gen_synthetic(64, 8, "clusters", rng_seed=1)
    return ref, (Q + np.float32(0.01))[:48]


def test_sweep_harness_files_match_reference(golden, tmp_path):
    """The sweep harness's host side against the live reference's run_sweep
    (evaluate.py:120-307): the ranges of generate_ranges, the GTC1 ground-truth
    files (SHA-256 key = file name, bytes) and the CSV header are the
    reference's byte for byte; the deterministic columns (recall,
    dist_evals_per_query) of the width-4 / 10-iteration cells follow from the
    oracle's search (a pinned restatement of searcher.py) scored by the
    product's recall_at_k."""
    from types import SimpleNamespace
    from oracle import beam, index_state as ist
    from paper_2604_16402_b200 import evaluate
    from paper_2604_16402_b200.datasets import generate_ranges, recall_at_k
    sw = golden("sweep")
    ref, Q = _sweep_inputs(golden)
    n = ref.count
    store = SimpleNamespace(X=ref.X[:n], scalars=ref.scalars[:n], count=n)
    cache = evaluate.GroundTruthCache(tmp_path)
    names = []
    rows = {tuple(r[:5]): r for r in sw["rows"]}
    for sel in SWEEP_SPEC["selectivities"]:
        ranges = generate_ranges(ref.scalars[:n], sel, len(Q), SWEEP_SPEC["rng_seed"])
        truth = [beam.exact_filtered(ref, q, 10, r.lower, r.upper)[0].astype(np.int64) for q, r in zip(Q, ranges)]
        key = cache._key(store, Q, 10, ranges, None)
        cache._write(tmp_path / f"{key}.gt", truth, 10)
        names.append(f"{key}.gt")
        rec, ev = [], []
        for i, (q, r) in enumerate(zip(Q, ranges)):
            res = beam.beam_search(ref, q, ist.SearchCfg(k=10, lower=r.lower, upper=r.upper, itopk=32, search_width=4,
                                                         max_iterations=10,
                                                         rng_seed=beam.derive_seed(SWEEP_SPEC["rng_seed"], i)))
            rec.append(recall_at_k(res.slots, truth[i], 10))
            ev.append(res.stats.dist_evals)
        want = rows[(sel, 10, 32, 4, 10)]
        assert float(np.nanmean(rec)) == want[5] and float(np.mean(ev)) == want[6], (sel, want)
    assert sorted(names) == list(sw["gt_names"])
    for i, name in enumerate(sw["gt_names"]):
        assert (tmp_path / name).read_bytes() == sw[f"gt_{i}"].tobytes()
        back = cache._read(tmp_path / name)
        assert all(t.dtype == np.int64 for t in back)
    evaluate.EvalReport().write_csv(tmp_path / "empty.csv")
    assert (tmp_path / "empty.csv").read_bytes() == sw["csv_header"].tobytes()


@pytest.mark.gpu
def test_run_sweep_matches_reference_rows(golden, tmp_path):
    """run_sweep over the reference-built small_index loaded into the device
    layout: every grid row's deterministic columns (recall, mean distance
    evaluations, SCC count) equal the reference's run_sweep, and the disk cache
    writes the reference's GTC1 files (names and bytes)."""
    import paper_2604_16402_b200 as g
    from paper_2604_16402_b200 import evaluate
    sw = golden("sweep")
    gold = golden("small")
    gi = g.load_index(gold["container"].tobytes(), g.BuildParams(k_max=16, k_local=8, bucket_capacity=250))
    _, Q = _sweep_inputs(golden)
    rep = evaluate.run_sweep(gi, Q, evaluate.SweepSpec(**SWEEP_SPEC), gt_cache=evaluate.GroundTruthCache(tmp_path))
    cols = list(sw["cols"])
    got = np.array([[r[c] for c in cols] for r in rep.rows], np.float64)
    assert got.shape == sw["rows"].shape
    assert np.array_equal(got, sw["rows"]), np.argwhere(got != sw["rows"])
    assert sorted(p.name for p in tmp_path.glob("*.gt")) == list(sw["gt_names"])
    for i, name in enumerate(sw["gt_names"]):
        assert (tmp_path / name).read_bytes() == sw[f"gt_{i}"].tobytes()
    rep.write_csv(tmp_path / "s.csv")
    assert (tmp_path / "s.csv").read_bytes().startswith(sw["csv_header"].tobytes())
