#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --config 5 --steps 20 --warmup 3 --no-cpu --no-pcg --no-sub --no-elastic > gpurun_out/r2l_c5.json 2> gpurun_out/r2l_c5.err
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "p31 or operators or cellwise or tagged" > gpurun_out/r2l_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_tests.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 1200 --launch-count 60 --csv --log-file gpurun_out/r2l_c5_smooth_launches.csv \
  python bench.py --config 5 --steps 3 --warmup 3 --no-cpu --no-pcg --no-sub --no-elastic > gpurun_out/r2l_ncu.log 2>&1
