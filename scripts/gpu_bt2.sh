mkdir -p gpurun_out/bt
for v in "" "FASTH_NO_PDL=1" "FASTH_BUILD2=1" "FASTH_BUILD2=1 FASTH_NO_PDL=1"; do
  echo "== $v"
  env $v FASTH_TRACE=gpurun_out/bt/t784 timeout 300 python scripts/trace_run.py 784 32 32 > gpurun_out/bt/run.log 2>&1
  python scripts/build_timeline.py gpurun_out/bt/t784.build.bin 25 | grep -v "block start"
done
