#!/bin/bash
# Direct top block: k_schur_form with direct-indexed tables staged by TMA (factor time, agreement with the full factorisation).
mkdir -p gpurun_out
timeout 900 python tools/direct_check.py > gpurun_out/r5c_direct_small.log 2>&1; echo "rc=$?" >> gpurun_out/r5c_direct_small.log
timeout 900 python tools/direct_check.py 5 > gpurun_out/r5c_direct_c5.log 2>&1; echo "rc=$?" >> gpurun_out/r5c_direct_c5.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5c_launches.csv python tools/op_launches.py 5,0,0 > gpurun_out/r5c_ncu.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_schur.py -q -m gpu -p no:cacheprovider > gpurun_out/r5c_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r5c_tests.log
