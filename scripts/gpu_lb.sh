#!/bin/bash
# Large-batch path: parity tests, config-5 timing (auto / forced chain path), kernel list.
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_lb.py -x -q --timeout 300 -s 2>&1 | tail -15
for m in 8192 2048; do
  timeout 120 python scripts/bench_config5.py --m-per-gpu $m
done
FASTH_LB=0 timeout 120 python scripts/bench_config5.py --m-per-gpu 2048
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/bench_config5.py --m-per-gpu 8192 --steps 1 --warmup 1 > gpurun_out/lb_launches.csv 2>&1
echo done
