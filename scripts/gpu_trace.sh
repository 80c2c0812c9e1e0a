mkdir -p gpurun_out/trace
FASTH_TRACE=gpurun_out/trace/t784 timeout 300 python scripts/trace_run.py 784 32 32 > gpurun_out/trace/run.log 2>&1
python scripts/trace_report.py gpurun_out/trace/t784.fwd.bin gpurun_out/trace/t784.bwd.bin > gpurun_out/trace/report.txt 2>&1
FASTH_TRACE=gpurun_out/trace/t2048 timeout 300 python scripts/trace_run.py 2048 32 32 >> gpurun_out/trace/run.log 2>&1
python scripts/trace_report.py gpurun_out/trace/t2048.fwd.bin >> gpurun_out/trace/report.txt 2>&1
cat gpurun_out/trace/report.txt
