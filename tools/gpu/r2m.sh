#!/bin/bash
mkdir -p gpurun_out
for cmp in 0 1 0 1; do
  for cfg in 3 5; do
    FDMGPU_COMPACT=$cmp timeout 900 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu --no-pcg --no-sub --no-elastic \
      >> gpurun_out/r2m_compact${cmp}_c${cfg}.json 2>> gpurun_out/r2m_compact${cmp}_c${cfg}.err
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "compact or operators" > gpurun_out/r2m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_tests.log
