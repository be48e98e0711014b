#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k 'regex:k_cells|k_gather|k_patch_gather|k_patch_solve' -c 18 --csv --log-file gpurun_out/r2p_c5_smooth.csv \
  python tools/op_repeat.py smooth 5,0,0 > gpurun_out/r2p_a.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k 'regex:k_cells|k_gather|k_quad' -c 20 --csv --log-file gpurun_out/r2p_c5_A.csv \
  python tools/op_repeat.py A 5,0,0 > gpurun_out/r2p_b.log 2>&1
