#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_schur.py -x -q -k "cholesky_top or c3" > gpurun_out/r3e_schur.log 2>&1; echo "rc=$?" >> gpurun_out/r3e_schur.log
for w in 4 8; do
  FDMGPU_SYMV_WARPS=$w timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-sub --no-elastic --no-pcg > gpurun_out/r3e_c5_w$w.json 2> gpurun_out/r3e_c5_w$w.err
  FDMGPU_SYMV_WARPS=$w timeout 600 python bench.py --config 3 --steps 20 --warmup 5 --no-cpu --no-elastic --no-pcg > gpurun_out/r3e_c3_w$w.json 2> gpurun_out/r3e_c3_w$w.err
done
