#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/cond_top.py 3 > gpurun_out/r3a_cond_c3.log 2>&1; echo "rc=$?" >> gpurun_out/r3a_cond_c3.log
timeout 1800 python tools/cond_top.py 5 > gpurun_out/r3a_cond_c5.log 2>&1; echo "rc=$?" >> gpurun_out/r3a_cond_c5.log
