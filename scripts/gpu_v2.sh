mkdir -p gpurun_out/v2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v2/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/v2/pytest_gpu.log
tail -30 gpurun_out/v2/pytest_gpu.log
FASTH_TRACE=gpurun_out/v2/t784 timeout 300 python scripts/trace_run.py 784 32 32 > gpurun_out/v2/trace_run.log 2>&1
python scripts/trace_report.py gpurun_out/v2/t784.*.bin > gpurun_out/v2/trace.txt 2>&1
cat gpurun_out/v2/trace.txt
timeout 600 python bench.py --steps 100 --no-cpu > gpurun_out/v2/bench.log 2>&1; tail -2 gpurun_out/v2/bench.log
