#!/bin/bash
# ncu --set full of k_schur_form2 (C5), with source; A/B factor time FDMGPU_FORM=1 vs default on the same box.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_schur_form2 -c 1 -o gpurun_out/r5m_form2 -f python tools/op_launches.py 5,0,0 > gpurun_out/r5m_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/r5m_ncu.log
for rep in 1 2; do
  timeout 300 python tools/factor_time.py 5,0,0 > gpurun_out/r5m_factor_form2_$rep.log 2>&1
  FDMGPU_FORM=1 timeout 300 python tools/factor_time.py 5,0,0 > gpurun_out/r5m_factor_form1_$rep.log 2>&1
done
