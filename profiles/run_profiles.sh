#!/bin/bash
# Round-1 profile capture (run on the GPU box via gpurun; outputs under gpurun_out/).
# Every ncu command is preceded by the identical command run plainly (&&), per the profiling recipe.
set -x
O=gpurun_out
python bench.py > $O/p_bench_default.json 2> $O/p_bench_default.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/launches_default.csv \
    python bench.py > $O/ncu_launch.log 2>&1
python bench.py --extra 0 --no-cpu --steps 2000 --warmup 50 > $O/p_c2.json 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_step_sw -s 1 -c 1 -o $O/prof_c2_sw \
    python bench.py --extra 0 --no-cpu --steps 2000 --warmup 50 > $O/ncu_c2.log 2>&1
python bench.py --config 3 --precision fp32 --steps 100 --warmup 3 --no-cpu --extra 0 > $O/p_c3f.json 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_wstep -s 3 -c 1 -o $O/prof_c3_fp32 \
    python bench.py --config 3 --precision fp32 --steps 100 --warmup 3 --no-cpu --extra 0 > $O/ncu_c3f.log 2>&1
# fp64 U-form k_ustep (configs 3 and 5): first launch (3 warm-up steps), one capture per gpurun call
python bench.py --config 3 --steps 20 --warmup 3 --no-cpu --extra 0 > $O/p3u.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_ustep -c 1 -o $O/ustep3 \
    python bench.py --config 3 --steps 20 --warmup 3 --no-cpu --extra 0 > $O/ncu3.log 2>&1
python bench.py --config 5 --steps 20 --warmup 3 --no-cpu --extra 0 > $O/p5b.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_ustep -c 1 -o $O/ustep5b \
    python bench.py --config 5 --steps 20 --warmup 3 --no-cpu --extra 0 > $O/ncu5b.log 2>&1
python bench.py --config 5 --steps 300 --warmup 5 --no-cpu --extra 0 > $O/b_c5.json 2>&1
python bench.py --config 5 --precision fp32 --steps 300 --warmup 5 --no-cpu --extra 0 > $O/b_c5f.json 2>&1
python bench.py --config 3 --precision fp32 --steps 300 --warmup 5 --no-cpu --extra 0 > $O/b_c3f.json 2>&1
ls -la $O
