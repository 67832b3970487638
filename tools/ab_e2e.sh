#!/bin/bash
# A/B the cfg2 bench's device and e2e numbers of prebuilt libraries: VARS="A B" bash tools/ab_e2e.sh [rounds]
cd "$(dirname "$0")/.."
L=paper_2604_16402_b200/libgrab.so
cp $L ab/lib_orig.so
for r in $(seq ${1:-2}); do
  for v in ${VARS:-A B}; do
    cp ab/lib$v.so $L
    echo "== $v round $r"
    python bench.py --no-sweep --no-cfg1 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['e2e_search_batch']['value'])"
  done
done
cp ab/lib_orig.so $L
