# A/B of env-knob variants at the metric config (fused and two-call) + GPU tests.
mkdir -p gpurun_out/ab
R=gpurun_out/ab
timeout 300 python scripts/step_env.py "$@" > $R/fused.jsonl 2> $R/fused.err
STEP_TWO_CALL=1 timeout 300 python scripts/step_env.py "$@" > $R/twocall.jsonl 2> $R/twocall.err
if [ -n "$AB_TESTS" ]; then timeout 900 python -m pytest tests -m gpu -q -x --timeout 240 $AB_TESTS > $R/pytest.log 2>&1; echo "exit $?" >> $R/pytest.log; tail -3 $R/pytest.log; fi
cat $R/fused.jsonl $R/twocall.jsonl; tail -3 $R/fused.err
