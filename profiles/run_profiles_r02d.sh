#!/bin/bash
# Round-2 (last session) profile of config 4 after the layer-0 pass moved into the sweep (k_step_mt):
# the TIMED 20-step launch (-s 1 skips the warm-up launch of the same kernel), after the same command
# has run plainly.
set -x
O=gpurun_out
B="--steps 20 --warmup 5 --no-cpu --extra 0"
python bench.py $B --config 4 > $O/p4.json 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_step_mt -s 1 -c 1 -o $O/r02_c4_mt2 \
    python bench.py $B --config 4 > $O/ncu_c4.log 2>&1
ls -la $O
