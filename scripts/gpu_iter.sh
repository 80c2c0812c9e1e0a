mkdir -p gpurun_out/it
timeout 900 python -m pytest tests -m gpu -x -q --timeout 240 > gpurun_out/it/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/it/pytest_gpu.log
tail -n 4 gpurun_out/it/pytest_gpu.log
timeout 120 python scripts/kernel_times.py 2>&1 | head -2
FASTH_TRACE=gpurun_out/it/b timeout 120 python scripts/trace_fused.py > /dev/null 2>&1; python scripts/trace_report.py gpurun_out/it/b.build.bin
timeout 300 python bench.py --steps 100 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print(l['value'], l['two_call_us_per_step'], l['e2e']['value'], l['kernel_us'], l['parity_max_rel_err'])"
