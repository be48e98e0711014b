#!/bin/bash
# Head evidence with the half-row-tile k_schur_form2: agreement with the full factorisation, default bench, reference arm, smoke, full GPU suite, C5 launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,power.limit --format=csv > gpurun_out/r5l_gpu.txt 2>&1
timeout 600 python tools/direct_check.py > gpurun_out/r5l_direct_small.log 2>&1; echo "rc=$?" >> gpurun_out/r5l_direct_small.log
timeout 600 python tools/direct_check.py 5 > gpurun_out/r5l_direct_c5.log 2>&1; echo "rc=$?" >> gpurun_out/r5l_direct_c5.log
FDMGPU_FORM=1 timeout 600 python tools/direct_check.py 5 > gpurun_out/r5l_direct_c5_form1.log 2>&1; echo "rc=$?" >> gpurun_out/r5l_direct_c5_form1.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r5l_bench.json 2> gpurun_out/r5l_bench.err; echo "rc=$?" >> gpurun_out/r5l_bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5l_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r5l_smoke.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r5l_ref.json 2> gpurun_out/r5l_ref.err; echo "rc=$?" >> gpurun_out/r5l_ref.err
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r5l_tests_all.log 2>&1; echo "rc=$?" >> gpurun_out/r5l_tests_all.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r5l_launches_c5.csv python tools/op_launches.py 5,0,0 > gpurun_out/r5l_ncu.log 2>&1
