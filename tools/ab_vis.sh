#!/bin/bash
# A/B ab/libA.so vs ab/libB.so on the search sweep points (alternating), then
# one DRAM-bytes ncu pass of each on the 10 % point.
cd "$(dirname "$0")/.."
L=paper_2604_16402_b200/libgrab.so
cp $L ab/lib_orig.so
PAIRS=${PAIRS:-0.01@400:4:150,0.1@296:4:100,0.5@464:4:150}
for r in 1 2; do
  for v in A B; do
    cp ab/lib$v.so $L
    echo "== $v round $r"; python tools/search_lab.py --config cfg2 --reps 10 --pairs $PAIRS 2>&1 | grep "stats="
  done
done
for v in A B; do
  cp ab/lib$v.so $L
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
      -k regex:k_search -s 2 -c 1 --csv python tools/search_lab.py --config cfg2 --reps 1 --pairs 0.1@296:4:100 \
      > gpurun_out/ab_vis_ncu_$v.csv 2>/dev/null
  echo "== ncu $v"; grep -E "dram__bytes|gpu__time|hit_rate" gpurun_out/ab_vis_ncu_$v.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
cp ab/lib_orig.so $L
