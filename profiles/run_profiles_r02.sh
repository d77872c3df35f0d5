#!/bin/bash
# Round-2 profile capture (run on the GPU box via gpurun; outputs under gpurun_out/).
# Every ncu command is preceded by the identical command run plainly (&&), per the profiling recipe;
# the captured launch is the TIMED one (-s skips the warm-up launch of the same kernel).
set -x
O=gpurun_out
B="--steps 20 --warmup 5 --no-cpu --extra 0"
# launch list of the headline command (config 5 fp64, headline only)
python bench.py $B > $O/p5.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_c5.csv \
    python bench.py $B > $O/ncu_l5.log 2>&1
# config 5 fp64 k_ustep, timed launch (#1; #0 is the warm-up run)
ncu --set full --import-source on --clock-control none -k regex:k_ustep -s 1 -c 1 -o $O/r02_c5_ustep \
    python bench.py $B > $O/ncu_c5.log 2>&1
# config 5 fp32 k_wstep: init + warm-up run, init + timed run -> launch #3
python bench.py $B --precision fp32 > $O/p5f.json 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_wstep -s 3 -c 1 -o $O/r02_c5f_wstep \
    python bench.py $B --precision fp32 > $O/ncu_c5f.log 2>&1
# config 3 fp64 k_ustep timed launch
python bench.py $B --config 3 > $O/p3.json 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_ustep -s 1 -c 1 -o $O/r02_c3_ustep \
    python bench.py $B --config 3 > $O/ncu_c3.log 2>&1
# config 2 k_step_sw timed launch (20 steps: includes the per-launch prologue)
python bench.py $B --config 2 > $O/p2.json 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_step_sw -s 1 -c 1 -o $O/r02_c2_sw \
    python bench.py $B --config 2 > $O/ncu_c2.log 2>&1
# ROM build: one k_pcg launch (config 3 recipe), one k_dgemm and one k_cholqr
ncu --set full --import-source on --clock-control none -k regex:k_pcg -s 3 -c 1 -o $O/r02_rom_pcg \
    python bench.py $B --config 3 > $O/ncu_pcg.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_dgemm -s 40 -c 1 -o $O/r02_rom_dgemm \
    python bench.py $B --config 3 > $O/ncu_dgemm.log 2>&1
# fine-grid FDTD (config 3 grid)
python bench.py --fdtd --config 3 --steps 20 --warmup 3 --no-cpu > $O/pf.json 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_fdtd -s 10 -c 1 -o $O/r02_fdtd \
    python bench.py --fdtd --config 3 --steps 20 --warmup 3 --no-cpu > $O/ncu_fdtd.log 2>&1
ls -la $O
