#!/bin/bash
# tools/ab_time.sh <script> rounds name... : interleaved runs of a timing script per library variant
script=$1; rounds=$2; shift 2
for r in $(seq $rounds); do for v in "$@"; do
  SFW_B200_LIB=build/ab/$v/libsfw_b200.so python $script 2>&1 | tail -1 >> gpurun_out/ab.txt
done; done
