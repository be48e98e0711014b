#!/bin/bash
mkdir -p gpurun_out
for v in "1 1" "0 1" "1 0" "0 0"; do
  set -- $v
  FDMGPU_COMP_STAGED=$1 FDMGPU_SPMV_STAGED=$2 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-sub --no-elastic --no-pcg > gpurun_out/r3r_c5_$1$2.json 2> gpurun_out/r3r_c5_$1$2.err
done
FDMGPU_COMP_STAGED=0 FDMGPU_SPMV_STAGED=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3r_launches_00.csv python tools/op_launches.py 5,0,0 > /dev/null 2>&1
