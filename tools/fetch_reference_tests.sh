#!/usr/bin/env bash
# Copy the reference package's own pytest suite (read-only /root/reference) into
# the git-ignored baseline/_ref_tests/, from where tests/test_gpu_reference_suite.py
# runs it on the GPU box against compat/bucketann (the drop-in alias). The copy
# travels with gpurun / the driver's snapshot like baseline/_ref; it is never
# committed.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${REFERENCE_TESTS:-/root/reference/pkg/tests}"
DST="$ROOT/baseline/_ref_tests"
[ -d "$SRC" ] || { echo "no reference tests at $SRC" >&2; exit 1; }
mkdir -p "$DST"
cp "$SRC"/*.py "$DST"/
ls "$DST"
