#!/bin/bash
# Head numbers of the four smaller configurations (DESIGN.md table), GPU legs only.
mkdir -p gpurun_out
for c in 1 2 3 4; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu --no-elastic > gpurun_out/r5p_c$c.json 2> gpurun_out/r5p_c$c.err; echo "rc=$?" >> gpurun_out/r5p_c$c.err
done
