#!/bin/bash
# ncu launch list of the bench command itself (C5 timed region: 3 warm-up + 3 steps; the CPU leg, PCG graph and sub-lines launch nothing inside it).
mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-pcg --no-sub --no-elastic > gpurun_out/r5o_bench_plain.json 2> gpurun_out/r5o_bench_plain.err; echo "rc=$?" >> gpurun_out/r5o_bench_plain.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r5o_bench_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu --no-pcg --no-sub --no-elastic > gpurun_out/r5o_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r5o_ncu.log
