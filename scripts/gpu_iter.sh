mkdir -p gpurun_out/it
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/it/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/it/pytest_gpu.log
tail -n 15 gpurun_out/it/pytest_gpu.log
python tools/fasth_bench_b200.py --d 256:256:4 --reps 20 --algo fasth,ref-fasth 2>&1 | tail -12
python tools/fasth_bench_b200.py --d 784 --reps 20 --op layer --k 32 2>&1 | tail -3
