#!/bin/bash
# A/B build time of two prebuilt libraries (ab/libA.so, ab/libB.so): bash tools/ab_build.sh cfg2 [rounds]
cd "$(dirname "$0")/.."
L=paper_2604_16402_b200/libgrab.so
cp $L ab/lib_orig.so
for r in $(seq ${2:-2}); do
  for v in ${VARS:-A B}; do
    cp ab/lib$v.so $L
    echo "== $v round $r"; python tools/build_lab.py --config ${1:-cfg2} --reps 3
  done
done
cp ab/lib_orig.so $L
