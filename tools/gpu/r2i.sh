#!/bin/bash
mkdir -p gpurun_out
for fu in 1 0; do
  for cfg in 5 3; do
    FDMGPU_FUSED=$fu timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-pcg --no-sub --no-elastic \
      > gpurun_out/r2i_fused${fu}_c${cfg}.json 2> gpurun_out/r2i_fused${fu}_c${cfg}.err
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "fused or not_spd" > gpurun_out/r2i_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_tests.log
timeout 900 python bench.py --elastic 3,8,15,1 --no-cpu --steps 20 --warmup 3 > gpurun_out/r2i_elastic.json 2> gpurun_out/r2i_elastic.err
