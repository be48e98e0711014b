#!/bin/bash
mkdir -p gpurun_out
for cfg in 3 5; do
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-pcg --no-sub --no-elastic \
    > gpurun_out/r2k_c${cfg}.json 2> gpurun_out/r2k_c${cfg}.err
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_state.py -x -q -m gpu > gpurun_out/r2k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_tests.log
