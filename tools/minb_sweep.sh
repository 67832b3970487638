#!/bin/bash
# Rebuild the search kernel with different register caps and time cfg2 search.
cd "$(dirname "$0")/.."
C=paper_2604_16402_b200/csrc
make -C $C -j16 >/dev/null
for MB in ${MINBS:-4 5 6}; do
  (cd $C && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
     --expt-relaxed-constexpr -DGRAB_SEARCH_MINB=$MB -c search.cu -o build/search.o && \
   nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../libgrab.so $(ls *.cu | sed 's/\.cu$/.o/; s/^/build\//'))
  echo "MINB=$MB"
  python tools/search_lab.py --config cfg2 --reps 10 --points "${POINTS:-224:4:100,128:4:50}" 2>&1 | grep -v "^ "
done
touch $C/search.cu
