# quick parity subset + A/B of env variants + build trace.  $AB_K selects tests (pytest -k)
mkdir -p gpurun_out/ab
R=gpurun_out/ab
timeout 600 python -m pytest tests/test_gpu_fasth.py tests/test_gpu_wy.py -q -x --timeout 240 ${AB_K:+-k "$AB_K"} > $R/pytest.log 2>&1; echo "exit $?" >> $R/pytest.log
tail -15 $R/pytest.log
timeout 300 python scripts/step_env.py "$@" > $R/fused.jsonl 2> $R/fused.err
STEP_TWO_CALL=1 timeout 300 python scripts/step_env.py "$@" > $R/twocall.jsonl 2> $R/twocall.err
cat $R/fused.jsonl $R/twocall.jsonl; tail -3 $R/fused.err
mkdir -p gpurun_out/bt
FASTH_TRACE=gpurun_out/bt/t784 timeout 300 python scripts/trace_run.py 784 32 32 > gpurun_out/bt/run.log 2>&1
python scripts/build_timeline.py gpurun_out/bt/t784.build.bin 25
