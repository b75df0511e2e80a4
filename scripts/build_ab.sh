#!/bin/bash
# Build an A/B variant of libcgvk.so with extra -D flags into build_ab/.
# usage: bash scripts/build_ab.sh name -DFLAG=V ...
set -eu
name=$1; shift
mkdir -p build_ab
R=$(cd "$(dirname "$0")/.." && pwd)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo --fmad=false \
  -Xcompiler -fPIC,-O2 -Xptxas -warn-spills -I "$R/include" "$@" -shared \
  -o "$R/build_ab/libcgvk_$name.so" "$R/paper_1905_01549_b200/csrc/cgvk_api.cu" -lcudart
echo "built build_ab/libcgvk_$name.so"
