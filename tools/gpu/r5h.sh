#!/bin/bash
# p = 31 slab transform T1: 8 vs 16 gathers in flight per thread (C5 step and S^T time).
mkdir -p gpurun_out
for b in 8 16 8 16; do FDMGPU_T1_BATCH=$b timeout 600 python bench.py --config 5 --steps 20 --warmup 5 --no-sub --no-cpu --no-pcg --no-elastic > gpurun_out/r5h_bench_b$b.json 2> gpurun_out/r5h_bench_b$b.err; python - <<PY >> gpurun_out/r5h_t1_ab.log
import json
d=json.loads(open('gpurun_out/r5h_bench_b$b.json').read().strip().splitlines()[-1])
print('T1_BATCH=$b step', d['ms_per_step'], 'S^T', d['transform_roofline']['ms'], 'solve', d['solve_roofline']['ms'], 'A', d['residual_roofline']['ms'])
PY
done
FDMGPU_T1_BATCH=16 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5.py -q -m gpu -k "p31 or slab" -p no:cacheprovider > gpurun_out/r5h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r5h_tests.log
