#!/bin/bash
# Schur-split solve: new tests, the parity suites, then C3 / C5 bench lines.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_schur.py -x -q > gpurun_out/r2u_schur.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_schur.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5.py -x -q > gpurun_out/r2u_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_parity.log
timeout 600 python bench.py --config 3 --steps 20 --warmup 5 --no-cpu --no-elastic > gpurun_out/r2u_c3.json 2> gpurun_out/r2u_c3.err; echo "rc=$?" >> gpurun_out/r2u_c3.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-sub --no-elastic > gpurun_out/r2u_c5.json 2> gpurun_out/r2u_c5.err; echo "rc=$?" >> gpurun_out/r2u_c5.err
