#!/bin/bash
# A/B a search-kernel compile flag on cfg2: bash tools/ab_search.sh "-DFLAG" [points]
cd "$(dirname "$0")/.."
C=paper_2604_16402_b200/csrc
make -C $C -j16 >/dev/null
P=${2:-304:4:100}
echo "== default"; python tools/search_lab.py --config cfg2 --reps 10 --points $P 2>&1 | grep "stats=False"
(cd $C && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
   --expt-relaxed-constexpr $1 -c search.cu -o build/search.o && \
 nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../libgrab.so build/*.o)
echo "== $1"; python tools/search_lab.py --config cfg2 --reps 10 --points $P 2>&1 | grep "stats=False"
touch $C/search.cu
