"""Anchor the reference arm's CPU port to the LIVE reference (lab tool, build
container only -- /root/reference does not exist on the GPU box).

bench.py --impl reference times oracle/beam.py (the numpy restatement of
searcher.py:156-233) because the reference is pure Python and cannot travel to
the box. This tool measures, on THIS host, single process, on one
reference-built graph:

* ``bucketann.search`` (the reference's own code path), and
* ``oracle.beam.beam_search`` (the port the reference arm runs),

for the same queries, ranges, parameters and per-query seeds, checks that
their results are identical (slots, f64 distances, every SearchStats counter),
and prints both rates and their ratio as one JSON line. The ratio converts the
box's port number into an estimate of the live reference's speed there.

    PYTHONPATH=/root/reference/pkg/src python tools/anchor_reference.py \
        > profiles/r02_reference_anchor.json
"""
from __future__ import annotations

import json
import os
import sys
import tempfile
import time

import numpy as np

import bucketann as ba
from bucketann.evaluate import generate_ranges
from bucketann.searcher import derive_query_seed

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import beam, index_state as ist  # noqa: E402
from paper_2604_16402_b200.datasets import gen_lowrank, lowrank_queries  # noqa: E402

N, D, CAP = int(os.environ.get("ANCHOR_N", 100_000)), 128, 6_250
NQ = int(os.environ.get("ANCHOR_NQ", 200))
OPS = {"cfg1_default": dict(k=10, itopk=128, search_width=4, max_iterations=50),
       "cfg2_r95": dict(k=10, itopk=296, search_width=4, max_iterations=100)}
STAT_KEYS = ["iterations", "dist_evals", "seed_evals", "gathered", "in_range_new", "precheck_rejected",
             "seed_attempts"]


def main():
    X, S = gen_lowrank(N, D, seed=0)
    t0 = time.perf_counter()
    index, _ = ba.build_index(X, S, ba.BuildParams(bucket_capacity=CAP))
    build_s = time.perf_counter() - t0
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "g.grab")
        ba.save_index(index, path)
        ref = ist.index_from_container(open(path, "rb").read())
    Q = lowrank_queries(NQ, D, seed=1)
    ranges = generate_ranges(index.store.scalars[:index.count], 0.1, NQ, 11)
    out = {"what": "live bucketann.search vs the oracle port (bench --impl reference) on one reference-built graph, "
                   "single process, same queries / ranges / seeds",
           "n": N, "dim": D, "bucket_capacity": CAP, "queries": NQ, "selectivity": 0.1,
           "reference_build_s": round(build_s, 1), "host_cpu": os.cpu_count(), "points": {}}
    for name, op in OPS.items():
        t0 = time.perf_counter()
        live = [ba.search(index, q, ba.SearchParams(range=r, rng_seed=derive_query_seed(11, i), **op))
                for i, (q, r) in enumerate(zip(Q, ranges))]
        t_live = time.perf_counter() - t0
        t0 = time.perf_counter()
        port = [beam.beam_search(ref, q, ist.SearchCfg(lower=r.lower, upper=r.upper, rng_seed=beam.derive_seed(11, i),
                                                      **op))
                for i, (q, r) in enumerate(zip(Q, ranges))]
        t_port = time.perf_counter() - t0
        same = all(np.array_equal(a.slots, b.slots) and np.array_equal(a.sq_dists, b.sq_dists)
                   and all(getattr(a.stats, k) == getattr(b.stats, k) for k in STAT_KEYS)
                   for a, b in zip(live, port))
        out["points"][name] = {**op, "reference_qps": round(NQ / t_live, 1), "port_qps": round(NQ / t_port, 1),
                               "port_over_reference": round(t_live / t_port, 3), "results_identical": same}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
