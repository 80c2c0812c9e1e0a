mkdir -p gpurun_out/bt
FASTH_TRACE=gpurun_out/bt/t784 timeout 300 python scripts/trace_run.py 784 32 32 > gpurun_out/bt/run.log 2>&1
ls gpurun_out/bt
python scripts/build_timeline.py gpurun_out/bt/t784.build.bin 25
