#!/bin/bash
# Full GPU suite, launch list + DRAM bytes of C5 / C3, --set full of the C5 top-block product.
mkdir -p gpurun_out
timeout 3000 python -m pytest tests/ -q -m gpu > gpurun_out/r3g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3g_tests.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r3g_launches_c5.csv python tools/op_launches.py 5,0,0 > gpurun_out/r3g_ncu_c5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r3g_launches_c3.csv python tools/op_launches.py 3,0,0 > gpurun_out/r3g_ncu_c3.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_schur_symv -s 1 -c 1 -o gpurun_out/r3g_symv python tools/op_launches.py 5,0,0 > gpurun_out/r3g_ncu_symv.log 2>&1
