#!/bin/bash
# CPU baseline matrix on the GPU box's host cores, then the C5 launch list.
mkdir -p gpurun_out
timeout 3000 python tools/cpu_baseline.py --configs 1,2,3,5 --reps 5 --out gpurun_out/r2d_cpu_baseline.json > gpurun_out/r2d_cpu_baseline.log 2>&1
echo "rc=$?" >> gpurun_out/r2d_cpu_baseline.log
lscpu > gpurun_out/r2d_lscpu.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2d_c5_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu --no-sub --no-elastic > gpurun_out/r2d_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2d_ncu.log
