#!/bin/bash
# Round-2 (late) profile capture for the kernels that replaced k_step_ms2 / k_step_sw:
# config 4 k_step_mt and config 2 k_step_sw4.  Each ncu command follows the same command run
# plainly; the captured launch is the TIMED one (-s skips the warm-up launch of the same kernel).
set -x
O=gpurun_out
B="--steps 20 --warmup 5 --no-cpu --extra 0"
python bench.py $B --config 4 > $O/p4.json 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_step_mt -s 1 -c 1 -o $O/r02_c4_mt \
    python bench.py $B --config 4 > $O/ncu_c4.log 2>&1
python bench.py $B --config 2 > $O/p2.json 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_step_sw -s 1 -c 1 -o $O/r02_c2_sw4 \
    python bench.py $B --config 2 > $O/ncu_c2.log 2>&1
ls -la $O
