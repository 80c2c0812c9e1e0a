# compute-sanitizer over the chain-path tests (builder v4, push-warp sweep, gradient kernel, host step)
mkdir -p gpurun_out/san
R=gpurun_out/san
echo "## memcheck: tests/test_gpu_fasth.py + tests/test_gpu_cpp.py" > $R/summary.txt
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_fasth.py tests/test_gpu_cpp.py -q -x > $R/memcheck.log 2>&1
grep -E "passed|failed" $R/memcheck.log | tail -1 >> $R/summary.txt; grep "ERROR SUMMARY" $R/memcheck.log | tail -1 >> $R/summary.txt
echo "## synccheck: golden / bitwise / build4 / host" >> $R/summary.txt
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_fasth.py -q -x -k "golden or bitwise or build4 or host" > $R/synccheck.log 2>&1
grep -E "passed|failed" $R/synccheck.log | tail -1 >> $R/summary.txt; grep "ERROR SUMMARY" $R/synccheck.log | tail -1 >> $R/summary.txt
echo "## racecheck: reference goldens cfg1 / ragged, fused and two-call" >> $R/summary.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_fasth.py -q -x -k "reference_golden and (cfg1 or ragged)" > $R/racecheck.log 2>&1
grep -E "passed|failed" $R/racecheck.log | tail -1 >> $R/summary.txt; grep "RACECHECK SUMMARY" $R/racecheck.log | tail -1 >> $R/summary.txt
cat $R/summary.txt
