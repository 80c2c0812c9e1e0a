#!/bin/bash
# LB path: tests, config-5 timing, launch list, ncu --set full of F1/F2 and the dV GEMM.
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_lb.py -x -q --timeout 300 -s 2>&1 | tail -10
timeout 120 python scripts/bench_config5.py --m-per-gpu 8192
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/bench_config5.py --m-per-gpu 8192 --steps 1 --warmup 1 > gpurun_out/lb_launches.csv 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 2 -o gpurun_out/lb_f1f2 -f python scripts/bench_config5.py --m-per-gpu 8192 --steps 1 --warmup 0 > gpurun_out/lb_ncu1.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel<1>" -c 1 -o gpurun_out/lb_dv -f python scripts/bench_config5.py --m-per-gpu 8192 --steps 1 --warmup 0 > gpurun_out/lb_ncu2.log 2>&1
echo done
