#!/bin/bash
# LB path profiling: launch list + ncu --set full of the aux kernels and one pair GEMM.
mkdir -p gpurun_out
B="python scripts/bench_config5.py --m-per-gpu 8192 --steps 1 --warmup 0"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv $B > gpurun_out/lb_launches.csv 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"q_reduce|tri_inv|dv_reduce" -c 3 -o gpurun_out/lb_aux -f $B > gpurun_out/lb_ncu_aux.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 2 -o gpurun_out/lb_pair -f $B > gpurun_out/lb_ncu_pair.log 2>&1
echo done
