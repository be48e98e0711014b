#!/bin/bash
mkdir -p gpurun_out
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/op_launches.py 3,0,0 > gpurun_out/r2x_c3_plain.log 2>&1; echo "rc=$?" >> gpurun_out/r2x_c3_plain.log
timeout 1500 python -m pytest tests/test_gpu_schur.py -x -q > gpurun_out/r2x_schur.log 2>&1; echo "rc=$?" >> gpurun_out/r2x_schur.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2x_launches_c3.csv python tools/op_launches.py 3,0,0 > gpurun_out/r2x_ncu_c3.log 2>&1
timeout 600 python bench.py --config 3 --steps 20 --warmup 5 --no-cpu --no-elastic > gpurun_out/r2x_c3.json 2> gpurun_out/r2x_c3.err; echo "rc=$?" >> gpurun_out/r2x_c3.err
