#!/bin/bash
# Round-2 GPU session A: FP64 peak probe (with clocks), new GPU tests, C5 bench, C5 solve traffic.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,temperature.gpu --format=csv > gpurun_out/r2a_smi.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/probe/fp64_peak.cu && \
  (nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/r2a_fp64_clocks.csv & SMI=$!; \
   /tmp/fp64_peak > gpurun_out/r2a_fp64_peak.txt 2>&1; kill $SMI)
timeout 2400 python -m pytest tests/test_gpu_state.py tests/test_gpu_c5.py -x -q -m gpu > gpurun_out/r2a_tests_new.log 2>&1
echo "new tests rc=$?" >> gpurun_out/r2a_tests_new.log
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
echo "bench rc=$?" >> gpurun_out/r2a_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:k_patch_solve -c 6 --csv --log-file gpurun_out/r2a_c5_solve_dram.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu --no-pcg --no-sub --no-elastic > gpurun_out/r2a_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2a_ncu.log
timeout 2400 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r2a_tests_parity.log 2>&1
echo "parity tests rc=$?" >> gpurun_out/r2a_tests_parity.log
