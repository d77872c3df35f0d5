#!/bin/bash
# Build a variant of the library with extra nvcc defines into build/<name>/libsfw.so
#   tools/build_variant.sh lwclk -DSFW_LW_CLK
set -e
name=$1; shift
out=build/$name; mkdir -p $out
for f in paper_1406_6923_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
     --expt-relaxed-constexpr "$@" -c $f -o $out/$b.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libsfw.so $out/*.o -lcudart
