#!/bin/bash
# Host-side AddressSanitizer build of libgrab (device code unchanged) for chasing
# host heap corruption: bash tools/asan_build.sh && LD_PRELOAD=$(gcc -print-file-name=libasan.so) \
#   ASAN_OPTIONS=protect_shadow_gap=0:detect_leaks=0 python ...
set -e
cd "$(dirname "$0")/../paper_2604_16402_b200/csrc"
mkdir -p build_asan
for f in *.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O1 -g -std=c++17 -Xcompiler -fPIC -Xcompiler -fsanitize=address \
    -Xcompiler -fno-omit-frame-pointer --expt-relaxed-constexpr -c $f -o build_asan/${f%.cu}.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -Xcompiler -fsanitize=address \
  -o ../libgrab.so build_asan/*.o
