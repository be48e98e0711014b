#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
  for v in old new; do
    if [ $v = old ]; then L="FDMGPU_LIB=$PWD/build_ab/paper_2107_14758_b200/lib/libfdmgpu.so"; else L="X=1"; fi
    for cfg in 3 5; do
      env $L timeout 900 python bench.py --config $cfg --steps 30 --warmup 3 --no-cpu --no-pcg --no-sub --no-elastic \
        >> gpurun_out/r2q_${v}_c${cfg}.json 2>> gpurun_out/r2q_${v}_c${cfg}.err
    done
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "operators or full_size_vectors" > gpurun_out/r2q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_tests.log
