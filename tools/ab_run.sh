#!/bin/bash
# Interleaved A/B timing of library variants (tools/ab_build.sh) with one bench command line:
#   tools/ab_run.sh "<bench args>" rounds name1 name2 ...  -> gpurun_out/ab.txt
args=$1; rounds=$2; shift 2
for r in $(seq $rounds); do
  for v in "$@"; do
    out=$(SFW_B200_LIB=build/ab/$v/libsfw_b200.so python bench.py $args 2>/dev/null | tail -1)
    echo "$v $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"])' 2>&1)" >> gpurun_out/ab.txt
  done
done
