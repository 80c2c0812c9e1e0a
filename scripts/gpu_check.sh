# Quick state check: GPU tests, smoke, bench line, launch list.  Outputs in gpurun_out/check/.
mkdir -p gpurun_out/check
R=gpurun_out/check
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $R/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 240 > $R/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $R/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $R/smoke.log 2>&1
timeout 600 python bench.py > $R/bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $R/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-config5 > $R/b_ncu.log 2>&1
tail -3 $R/pytest_gpu.log; tail -2 $R/bench.log
