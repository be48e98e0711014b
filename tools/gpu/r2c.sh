#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sipg.py -x -q -m gpu > gpurun_out/r2c_sipg.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_sipg.log
