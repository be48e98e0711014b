#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_smoke.log
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err; echo "rc=$?" >> gpurun_out/r2s_bench.err
timeout 1800 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2s_ref.json 2> gpurun_out/r2s_ref.err; echo "rc=$?" >> gpurun_out/r2s_ref.err
