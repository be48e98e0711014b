#!/bin/bash
# Compact solve records + panel-only factor operand loads: A/B timing and parity.
mkdir -p gpurun_out
for cfg in 3 5; do
  for cmp in 0 1; do
    FDMGPU_COMPACT=$cmp timeout 900 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu --no-pcg --no-sub --no-elastic \
      > gpurun_out/r2e_bench_c${cfg}_compact${cmp}.json 2> gpurun_out/r2e_bench_c${cfg}_compact${cmp}.err
  done
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_state.py tests/test_gpu_sipg.py -x -q -m gpu > gpurun_out/r2e_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_tests.log
timeout 900 python -m pytest tests/test_gpu_c5.py -x -q -m gpu > gpurun_out/r2e_tests_c5.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_tests_c5.log
