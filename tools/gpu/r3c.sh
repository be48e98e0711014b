#!/bin/bash
# Default bench (C5 headline + C3 / elasticity / SIPG sub-lines + CPU leg), then a
# --set full capture of the C5 top-block product and the coupling kernels.
mkdir -p gpurun_out
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r3c_bench.json 2> gpurun_out/r3c_bench.err; echo "rc=$?" >> gpurun_out/r3c_bench.err
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_schur_symv -s 1 -c 1 -o gpurun_out/r3c_symv python tools/op_launches.py 5,0,0 > gpurun_out/r3c_ncu_symv.log 2>&1; echo "rc=$?" >> gpurun_out/r3c_ncu_symv.log
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_schur_spmv|k_schur_comp" -s 4 -c 4 -o gpurun_out/r3c_sparse python tools/op_launches.py 5,0,0 > gpurun_out/r3c_ncu_sparse.log 2>&1; echo "rc=$?" >> gpurun_out/r3c_ncu_sparse.log
