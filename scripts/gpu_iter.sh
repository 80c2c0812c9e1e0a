mkdir -p gpurun_out/it
timeout 900 python -m pytest tests -m gpu -x -q --timeout 240 > gpurun_out/it/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/it/pytest_gpu.log
tail -n 4 gpurun_out/it/pytest_gpu.log
timeout 120 python scripts/e2e_breakdown.py
