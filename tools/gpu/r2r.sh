#!/bin/bash
mkdir -p gpurun_out
timeout 3000 python -m pytest tests/ -q -m gpu > gpurun_out/r2r_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_tests.log
