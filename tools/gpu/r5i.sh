#!/bin/bash
# p = 31 relaxation: boundary-only S^T gather + cell-local interior right-hand side (FDMGPU_SMOOTH_LOCAL) A/B, parity.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_c5.py -q -m gpu -x -p no:cacheprovider > gpurun_out/r5i_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r5i_tests.log
for m in 0 1 0 1; do FDMGPU_SMOOTH_LOCAL=$m timeout 600 python bench.py --config 5 --steps 20 --warmup 5 --no-sub --no-cpu --no-pcg --no-elastic > gpurun_out/r5i_bench_l$m.json 2> gpurun_out/r5i_bench_l$m.err; python - <<PY >> gpurun_out/r5i_local_ab.log
import json
d=json.loads(open('gpurun_out/r5i_bench_l$m.json').read().strip().splitlines()[-1])
print('SMOOTH_LOCAL=$m step', d['ms_per_step'], 'GDOF/s', d['value'], 'e2e', d['e2e']['value'], 'solve', d['solve_roofline']['ms'])
PY
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r5i_launches_c5.csv python tools/op_launches.py 5,0,0 > gpurun_out/r5i_ncu_c5.log 2>&1
