#!/bin/bash
# Residual kernels: mode 3 (stage 2 / 3 outputs over their inputs: more CTAs per SM) against mode 2; parity.
mkdir -p gpurun_out
for m in 2 3; do FDMGPU_QUAD_STRIP=$m timeout 300 python tools/quad_ab.py 5,0,0 >> gpurun_out/r5f_quad_ab.log 2>&1; done
for m in 2 3; do FDMGPU_QUAD_STRIP=$m timeout 300 python tools/quad_ab.py 5,4,7 >> gpurun_out/r5f_quad_ab.log 2>&1; done
FDMGPU_QUAD_STRIP=3 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5.py -q -m gpu -k "quad or p31 or trilinear or slab" -p no:cacheprovider > gpurun_out/r5f_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r5f_tests.log
FDMGPU_QUAD_STRIP=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5f_launches.csv python tools/op_launches.py 5,0,0 A > gpurun_out/r5f_ncu.log 2>&1
# coupling products: 8 vs 16 threads per row (C5 step, solve class)
for t in 8 16; do FDMGPU_SPMV_TPR=$t timeout 600 python bench.py --config 5 --steps 20 --warmup 5 --no-sub --no-cpu --no-pcg --no-elastic > gpurun_out/r5f_bench_tpr$t.json 2> gpurun_out/r5f_bench_tpr$t.err; done
FDMGPU_SPMV_TPR=16 timeout 600 python -m pytest tests/test_gpu_schur.py -q -m gpu -p no:cacheprovider > gpurun_out/r5f_tests_tpr16.log 2>&1; echo "rc=$?" >> gpurun_out/r5f_tests_tpr16.log
