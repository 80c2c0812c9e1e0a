mkdir -p gpurun_out/it
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/it/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/it/pytest_gpu.log
tail -n 3 gpurun_out/it/pytest_gpu.log
python scripts/kernel_times.py 2>&1 | head -1
FASTH_TRACE=gpurun_out/it/t784 timeout 300 python scripts/trace_run.py 784 32 32 > gpurun_out/it/trace_run.log 2>&1
python scripts/trace_report.py gpurun_out/it/t784.build.bin
