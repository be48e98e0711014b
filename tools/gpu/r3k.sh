#!/bin/bash
# Per-config bench lines (C1..C5) after the Schur split, plus elasticity / SIPG lines.
mkdir -p gpurun_out
for c in 1 2 4; do
  timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu --no-elastic > gpurun_out/r3k_c$c.json 2> gpurun_out/r3k_c$c.err
done
timeout 900 python bench.py --elastic 3,8,15,1 --steps 20 --warmup 5 --no-cpu > gpurun_out/r3k_el.json 2> gpurun_out/r3k_el.err
timeout 600 python bench.py --sipg 3,4,5 --steps 20 --warmup 5 --no-cpu > gpurun_out/r3k_sipg.json 2> gpurun_out/r3k_sipg.err
