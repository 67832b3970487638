#!/bin/bash
# A/B two prebuilt libgrab.so files (ab/libA.so, ab/libB.so) on one box, alternating:
#   bash tools/ab_lib.sh "cfg2:296:4:100 cfg3:328:4:100" [rounds]
cd "$(dirname "$0")/.."
L=paper_2604_16402_b200/libgrab.so
cp $L ab/lib_orig.so
for r in $(seq ${2:-2}); do
  for v in ${VARS:-A B}; do
    cp ab/lib$v.so $L
    for cp_ in $1; do
      cfg=${cp_%%:*}; pt=${cp_#*:}
      echo "== $v round $r $cfg"; python tools/search_lab.py --config $cfg --reps 10 --points $pt 2>&1 | grep "stats="
    done
  done
done
cp ab/lib_orig.so $L
