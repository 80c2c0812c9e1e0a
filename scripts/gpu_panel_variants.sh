#!/bin/bash
# Panel-kernel tuning variants (lib/variants/*.so, FASTH_LIB) on config 5 + parity.
set -x
mkdir -p gpurun_out
for lib in paper_2009_13977_b200/lib/libfasth_b200.so paper_2009_13977_b200/lib/variants/*.so; do
  echo "== $lib"
  FASTH_LIB=$lib timeout 120 python scripts/bench_config5.py --m-per-gpu 8192
  FASTH_LIB=$lib timeout 120 python scripts/bench_config5.py --m-per-gpu 1024
  FASTH_LIB=$lib timeout 240 python -m pytest tests -m gpu -k panel -x -q --timeout 200 2>&1 | tail -2
done
timeout 300 python scripts/bench_configs.py 2>&1 | tail -8
