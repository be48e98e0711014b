#!/bin/bash
# ncu --set full of k_schur_form (C5), with source.
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_schur_form -c 1 -o gpurun_out/r5d_form -f python tools/op_launches.py 5,0,0 > gpurun_out/r5d_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/r5d_ncu.log
