#!/bin/bash
# Build tuning variants of the CUDA library into variants/ (git-ignored .so
# files travel to the GPU box).  Usage: tools/build_variants.sh NAME "-DFLAG=V ..." ...
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode=arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Iinclude -Xcompiler -fPIC -shared $flags -o variants/lib_$name.so \
    paper_1708_01135_b200/csrc/ewald_b200.cu &
done
wait
ls variants
