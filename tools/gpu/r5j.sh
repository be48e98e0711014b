#!/bin/bash
# Final head evidence of round 2: smoke, default bench, reference arm, C5 launch list, symv --set full, full GPU suite.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,power.limit --format=csv > gpurun_out/r5j_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5j_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r5j_smoke.log
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r5j_bench.json 2> gpurun_out/r5j_bench.err; echo "rc=$?" >> gpurun_out/r5j_bench.err
timeout 1800 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r5j_ref.json 2> gpurun_out/r5j_ref.err; echo "rc=$?" >> gpurun_out/r5j_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r5j_launches_c5.csv python tools/op_launches.py 5,0,0 > gpurun_out/r5j_ncu_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_schur_symv -c 1 -o gpurun_out/r5j_symv -f python tools/op_launches.py 5,0,0 > gpurun_out/r5j_ncu_symv.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r5j_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r5j_tests.log
