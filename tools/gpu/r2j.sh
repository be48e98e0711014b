#!/bin/bash
# ncu --set full captures of the cell kernels (residual and basis transforms), one launch each.
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on -c 1"
timeout 600 $N -k regex:k_cells_stiffness16 -o gpurun_out/r2j_stiff16 python tools/op_repeat.py A 3,0,0 > gpurun_out/r2j_a.log 2>&1
timeout 600 $N -k regex:k_cells_transform16 -o gpurun_out/r2j_tr16 python tools/op_repeat.py St 3,0,0 > gpurun_out/r2j_b.log 2>&1
timeout 600 $N -k regex:k_cells_t1_32 -o gpurun_out/r2j_t1_32 python tools/op_repeat.py St 5,4,31 > gpurun_out/r2j_c.log 2>&1
timeout 600 $N -k regex:k_cells_t2_32 -o gpurun_out/r2j_t2_32 python tools/op_repeat.py St 5,4,31 > gpurun_out/r2j_d.log 2>&1
timeout 600 $N -k regex:k_quad_stage2 -o gpurun_out/r2j_quad2 python tools/op_repeat.py A 5,4,31 > gpurun_out/r2j_e.log 2>&1
ls -la gpurun_out/r2j_*
