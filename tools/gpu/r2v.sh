#!/bin/bash
# Launch lists (gpu__time_duration) of C3 and C5: factor + 2 smooth + 2 apply_A.
mkdir -p gpurun_out
for cfg in 3,0,0 5,0,0; do
  tag=${cfg%%,*}
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2v_launches_c$tag.csv python tools/op_launches.py $cfg > gpurun_out/r2v_ncu_c$tag.log 2>&1
  echo "rc=$?" >> gpurun_out/r2v_ncu_c$tag.log
done
