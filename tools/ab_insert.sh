#!/bin/bash
# A/B insert phase timings of prebuilt libraries ab/lib{A,B,...}.so: VARS="A B" bash tools/ab_insert.sh [rounds]
cd "$(dirname "$0")/.."
L=paper_2604_16402_b200/libgrab.so
cp $L ab/lib_orig.so
for r in $(seq ${1:-2}); do
  for v in ${VARS:-A B}; do
    cp ab/lib$v.so $L
    echo "== $v round $r"; python tools/profile_insert.py | grep "^insert" | grep -o "phase_seconds.*"
  done
done
cp ab/lib_orig.so $L
