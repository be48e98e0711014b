#!/bin/bash
# ncu --set full of the fused factor kernel: a heavy (K = 28) and a middle (K = 16) tile column at C3.
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on -k regex:k_patch_column -c 1"
timeout 900 $N --launch-skip 16 -o gpurun_out/r2n_col_heavy python tools/factor_time.py 3,0,0 > gpurun_out/r2n_a.log 2>&1
timeout 900 $N --launch-skip 4 -o gpurun_out/r2n_col_mid python tools/factor_time.py 3,0,0 > gpurun_out/r2n_b.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_patch -c 40 --csv --log-file gpurun_out/r2n_c3_factor_launches.csv python tools/factor_time.py 3,0,0 > gpurun_out/r2n_c.log 2>&1
ls -la gpurun_out/r2n_*
