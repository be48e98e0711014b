#!/bin/bash
# Residual (trilinear quadrature) kernels: row-strip DMMA tasks A/B (0 = 8x16 tasks, 1 / 2 = strips, k unrolled 2 / 4), parity.
mkdir -p gpurun_out
for m in 0 1 2; do FDMGPU_QUAD_STRIP=$m timeout 300 python tools/quad_ab.py 5,0,0 >> gpurun_out/r5b_quad_ab.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5.py -q -m gpu -k "quad or p31 or trilinear or slab" -p no:cacheprovider > gpurun_out/r5b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r5b_tests.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5b_launches.csv python tools/op_launches.py 5,0,0 A > gpurun_out/r5b_ncu.log 2>&1
