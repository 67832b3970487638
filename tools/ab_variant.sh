#!/bin/bash
# Build a libgrab.so variant into ab/lib$1.so from the current tree with extra
# nvcc flags for one source (default search.cu), reusing the other objects:
#   bash tools/ab_variant.sh C "-DGRAB_VIS_NO_DISCARD" [search.cu] [src-file-override]
set -e
cd "$(dirname "$0")/../paper_2604_16402_b200/csrc"
V=$1; FLAGS=$2; SRC=${3:-search.cu}; IN=${4:-$SRC}
mkdir -p ../../ab build/ab$V
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr"
$NV $FLAGS -I. -c $IN -o build/ab$V/${SRC%.cu}.o
OBJS=$(ls build/*.o | grep -v "/${SRC%.cu}.o$")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../../ab/lib$V.so $OBJS build/ab$V/${SRC%.cu}.o -Xcompiler -fvisibility=hidden
echo "ab/lib$V.so"
