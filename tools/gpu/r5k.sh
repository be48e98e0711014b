#!/bin/bash
# Direct top block: half-row-tile k_schur_form2 (double-buffered Y) -- agreement with the full factorisation, factor time, launch list, Schur tests.
mkdir -p gpurun_out
timeout 900 python tools/direct_check.py > gpurun_out/r5k_direct_small.log 2>&1; echo "rc=$?" >> gpurun_out/r5k_direct_small.log
timeout 900 python tools/direct_check.py 5 > gpurun_out/r5k_direct_c5.log 2>&1; echo "rc=$?" >> gpurun_out/r5k_direct_c5.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5k_launches.csv python tools/op_launches.py 5,0,0 > gpurun_out/r5k_ncu.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_schur.py -q -m gpu -p no:cacheprovider > gpurun_out/r5k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r5k_tests.log
# head evidence with the half-row-tile form kernel: default bench, reference arm, full GPU suite
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r5k_bench.json 2> gpurun_out/r5k_bench.err; echo "rc=$?" >> gpurun_out/r5k_bench.err
timeout 1800 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r5k_ref.json 2> gpurun_out/r5k_ref.err; echo "rc=$?" >> gpurun_out/r5k_ref.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5k_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r5k_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r5k_tests_all.log 2>&1; echo "rc=$?" >> gpurun_out/r5k_tests_all.log
