#!/bin/bash
# Full GPU suite + default bench + smoke (the driver's round-end sequence).
mkdir -p gpurun_out
timeout 3000 python -m pytest tests/ -q -m gpu > gpurun_out/r2t_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2t_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_smoke.log
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err; echo "rc=$?" >> gpurun_out/r2t_bench.err
