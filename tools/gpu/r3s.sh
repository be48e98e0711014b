#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_c5.py tests/test_gpu_schur.py -x -q > gpurun_out/r3s_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3s_tests.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r3s_launches_c5.csv python tools/op_launches.py 5,0,0 > gpurun_out/r3s_ncu_c5.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-sub --no-elastic --no-pcg > gpurun_out/r3s_c5.json 2> gpurun_out/r3s_c5.err
