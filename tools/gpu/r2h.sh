#!/bin/bash
# A/B: fused tile-column factorisation (k_patch_column) vs separate update / trsm launches.
mkdir -p gpurun_out
for fu in 0 1; do
  for cfg in 3 5; do
    FDMGPU_FUSED=$fu timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-pcg --no-sub --no-elastic \
      > gpurun_out/r2h_fused${fu}_c${cfg}.json 2> gpurun_out/r2h_fused${fu}_c${cfg}.err
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "fused or compact or not_spd or operators" > gpurun_out/r2h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_tests.log
