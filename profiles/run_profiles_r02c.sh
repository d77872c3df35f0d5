#!/bin/bash
# Round-2 (last session) profile capture for the kernels that had no ncu summary yet: the ROM
# build's k_pcg2 (DMMA line passes), k_cholqr, k_sfraction, k_stencil, the band LU k_gb_ntd, and
# the stepping instance of k_fdtd.  Each ncu command follows the same command run plainly.
set -x
O=gpurun_out
python tools/rom_time.py 3 > $O/rom3.json 2>&1 || exit 1
for spec in "k_pcg2 3" "k_cholqr 2" "k_sfraction 0" "k_stencil 1"; do
  set -- $spec
  ncu --set full --import-source on --clock-control none -k regex:$1 -s $2 -c 1 -o $O/r02_rom_$1 \
      python tools/rom_time.py 3 > $O/ncu_$1.log 2>&1
done
python tools/ntd_bench.py > $O/ntd.json 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_gb_ntd -s 1 -c 1 -o $O/r02_gb_ntd \
    python tools/ntd_bench.py > $O/ncu_ntd.log 2>&1
python bench.py --fdtd --config 3 --steps 20 --warmup 3 --no-cpu > $O/fdtd.json 2>&1 && \
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:k_fdtd<\(int\)0>' -s 30 -c 1 \
    -o $O/r02_fdtd0 python bench.py --fdtd --config 3 --steps 20 --warmup 3 --no-cpu > $O/ncu_fdtd0.log 2>&1
# (the stepping kernel k_fdtd<0>; an unqualified -k k_fdtd lands on k_fdtd<2>, the operator product of the CFL
#  power iteration, which is what profiles/r02_fdtd.txt holds)
ls -la $O
