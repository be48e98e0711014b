#!/bin/bash
# compute-sanitizer (memcheck, racecheck) on small cases that run this session's kernels: direct top block
# (k_schur_form with TMA-staged tables), residual GEMM variants (register-held outputs stored over the input).
mkdir -p gpurun_out
which compute-sanitizer > gpurun_out/r5g_sanitizer.log 2>&1
for tool in memcheck racecheck; do
  echo "== $tool 4,2,7 (factor + smooth + A) ==" >> gpurun_out/r5g_sanitizer.log
  timeout 900 compute-sanitizer --tool $tool python tools/op_launches.py 4,2,7 >> gpurun_out/r5g_sanitizer.log 2>&1; echo "rc=$?" >> gpurun_out/r5g_sanitizer.log
  echo "== $tool 5,2,5 (trilinear residual) ==" >> gpurun_out/r5g_sanitizer.log
  timeout 900 compute-sanitizer --tool $tool python tools/op_launches.py 5,2,5 A >> gpurun_out/r5g_sanitizer.log 2>&1; echo "rc=$?" >> gpurun_out/r5g_sanitizer.log
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "quadrature_gemm_task" -p no:cacheprovider > gpurun_out/r5g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r5g_tests.log
