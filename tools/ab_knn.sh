#!/bin/bash
# A/B the kNN screen time (GRAB_DEBUG timers) of prebuilt ab/lib*.so on cfg2 builds: VARS="A B" bash tools/ab_knn.sh
cd /root/repo
L=paper_2604_16402_b200/libgrab.so
cp $L ab/lib_orig.so
for r in 1 2; do for v in ${VARS:-A B}; do cp ab/lib$v.so $L; echo "== $v $r"; GRAB_DEBUG=1 python tools/build_lab.py --config cfg2 --reps 2 2>&1 | grep "knn jobs" | tail -2; done; done
cp ab/lib_orig.so $L 2>/dev/null || true
