#!/bin/bash
# Round-2 GPU session B: SIPG-DG device path tests, layout refactor regression (CG parity), C++ consumer.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sipg.py -x -q -m gpu > gpurun_out/r2b_sipg.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_sipg.log
timeout 600 python -m pytest tests/test_capi_consumer.py -x -q -m gpu > gpurun_out/r2b_consumer.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_consumer.log
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_elasticity.py -x -q -m gpu > gpurun_out/r2b_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_parity.log
