"""CPU oracle for the GRAB-ANNS range-filtered graph index -- TEST INFRASTRUCTURE.

This package restates, in numpy, the reference algorithm that
paper_2604_16402_b200 re-implements in CUDA (reference: /root/reference/pkg,
the pure-Python ``bucketann`` package; numpy 2.3.5 is the pinned third-party
dependency whose RNG/sort/GEMM semantics it relies on).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import it, and only as the checker or the timed CPU baseline. The
product path (paper_2604_16402_b200) never imports it and fails loudly when its
CUDA library is missing.

Parity pinning: tests/golden/*.npz were produced by running the live reference
(tests/golden/make_golden.py, PYTHONPATH=/root/reference/pkg/src) and
tests/test_oracle_golden.py checks this restatement against every vector.
"""
from . import beam, construct, index_state, ingest, rng  # noqa: F401
