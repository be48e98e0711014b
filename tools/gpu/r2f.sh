#!/bin/bash
# A/B: solve kernel with compact records (branch-free main pass + compact tails) vs the pre-compact library.
mkdir -p gpurun_out
run() {  # label, env...
  local label=$1; shift
  for cfg in 3 5; do
    env "$@" timeout 900 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu --no-pcg --no-sub --no-elastic \
      > gpurun_out/r2f_${label}_c${cfg}.json 2> gpurun_out/r2f_${label}_c${cfg}.err
  done
}
run old FDMGPU_LIB=$PWD/build_ab/paper_2107_14758_b200/lib/libfdmgpu.so
run compact1 FDMGPU_COMPACT=1
run compact0 FDMGPU_COMPACT=0
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "operators or full_size_vectors or cluster or inplace" > gpurun_out/r2f_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_tests.log
