#!/bin/bash
# Schur split v2 kernels: tests, launch lists, C3/C5 bench lines.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_schur.py -x -q > gpurun_out/r3b_schur.log 2>&1; echo "rc=$?" >> gpurun_out/r3b_schur.log
for cfg in 3,0,0 5,0,0; do
  tag=${cfg%%,*}
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3b_launches_c$tag.csv python tools/op_launches.py $cfg > gpurun_out/r3b_ncu_c$tag.log 2>&1
  echo "rc=$?" >> gpurun_out/r3b_ncu_c$tag.log
done
timeout 600 python bench.py --config 3 --steps 20 --warmup 5 --no-cpu --no-elastic > gpurun_out/r3b_c3.json 2> gpurun_out/r3b_c3.err; echo "rc=$?" >> gpurun_out/r3b_c3.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-sub --no-elastic > gpurun_out/r3b_c5.json 2> gpurun_out/r3b_c5.err; echo "rc=$?" >> gpurun_out/r3b_c5.err
