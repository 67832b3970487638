#!/bin/bash
# A/B prebuilt libgrab.so variants (ab/lib{A,B,...}.so) on cfg2 over selectivity@point pairs:
#   VARS="A B C" bash tools/ab_lib_pairs.sh "0.1@296:4:100,0.01@400:4:150" [rounds]
cd "$(dirname "$0")/.."
L=paper_2604_16402_b200/libgrab.so
cp $L ab/lib_orig.so
for r in $(seq ${2:-2}); do
  for v in ${VARS:-A B}; do
    cp ab/lib$v.so $L
    echo "== $v round $r"; python tools/search_lab.py --config cfg2 --reps 10 --pairs "$1" 2>&1 | grep "stats=False"
  done
done
cp ab/lib_orig.so $L
