#!/bin/bash
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_cells_t1_32|k_cells_t2_32|k_gather|k_schur_spmv|k_schur_comp" -s 10 -c 8 -o gpurun_out/r3n_cells python tools/op_launches.py 5,0,0 > gpurun_out/r3n_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/r3n_ncu.log
