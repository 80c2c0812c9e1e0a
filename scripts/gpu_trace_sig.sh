# Per-warp sweep traces of the two-call step, serial vs pipelined gradient (tape-warp sweep).
mkdir -p gpurun_out/tsig
for v in 0 1; do
  FASTH_DV_PIPE=$v FASTH_TRACE=gpurun_out/tsig/p$v timeout 300 python scripts/trace_run.py 784 32 32 > gpurun_out/tsig/run$v.log 2>&1
  ls gpurun_out/tsig/ >> gpurun_out/tsig/run$v.log
  python scripts/trace_report.py gpurun_out/tsig/p$v.bwd.v2.bin gpurun_out/tsig/p$v.bwd.warps.bin > gpurun_out/tsig/report$v.txt 2>&1
done
cat gpurun_out/tsig/report0.txt gpurun_out/tsig/report1.txt
