#!/bin/bash
# Build variants of libsfw_b200.so that differ only in compile-time knobs of one source file, for
# A/B timing on one GPU box:  tools/ab_build.sh <src.cu> <name> "<-D flags>" ...
# output: build/ab/<name>/libsfw_b200.so (the other objects are the default build's)
set -e
src=$1; shift
base=$(basename $src .cu)
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  mkdir -p build/ab/$name
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr $flags \
    -c $src -o build/ab/$name/$base.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/ab/$name/libsfw_b200.so \
    $(ls build/*.o | grep -v "build/$base.o") build/ab/$name/$base.o -lcudart
done
