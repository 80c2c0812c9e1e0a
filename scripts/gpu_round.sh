# Round evidence: GPU parity tests, bench (+ reference arm), launch list and
# ncu --set full of each kernel, secondary configs.  Outputs in gpurun_out/round/.
set -x
mkdir -p gpurun_out/round
R=gpurun_out/round
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $R/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 240 > $R/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $R/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $R/smoke.log 2>&1
timeout 600 python bench.py > $R/bench.log 2>&1
timeout 300 python bench.py --impl reference --steps 10 --warmup 3 > $R/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $R/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > $R/b_ncu.log 2>&1
for k in sweep2 build4 dv2; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 20 -c 1 -o $R/${k}_full python bench.py --steps 2 --warmup 3 --no-cpu > $R/ncu_$k.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:panel -s 2 -c 1 -o $R/panel_full python scripts/bench_config5.py --m-per-gpu 1024 --steps 1 --warmup 1 > $R/ncu_panel.log 2>&1
for m in 1024 8192; do timeout 300 python scripts/bench_config5.py --m-per-gpu $m --steps 3 --warmup 1 >> $R/config5.log 2>&1; done
timeout 900 python scripts/bench_configs.py > $R/configs.log 2>&1
timeout 300 python tools/fasth_bench_b200.py --d 256:256:4 --reps 20 --algo fasth,ref-fasth > $R/cli_mul.csv 2>&1
ls -la $R
mkdir -p gpurun_out/round/st
FASTH_STEPTRACE=gpurun_out/round/st/t timeout 300 python scripts/step_trace_run.py > gpurun_out/round/timeline.txt 2>&1
FASTH_STEPTRACE=gpurun_out/round/st/e timeout 300 python scripts/e2e_trace.py >> gpurun_out/round/timeline.txt 2>&1
FASTH_TRACE=gpurun_out/round/st/f timeout 300 python scripts/trace_fused.py 784 32 32 > /dev/null 2>&1
python scripts/trace_report.py "gpurun_out/round/st/f.sweep(fwd+bwd).v2.bin" "gpurun_out/round/st/f.sweep(fwd+bwd).warps.bin" > gpurun_out/round/sweep_trace.txt 2>&1
python scripts/build_timeline.py gpurun_out/round/st/f.build.bin 25 > gpurun_out/round/build_timeline.txt 2>&1
timeout 300 python scripts/replay_overhead.py > gpurun_out/round/replay_overhead.txt 2>&1
timeout 300 python scripts/e2e_ab.py base FASTH_D2H=dma > gpurun_out/round/e2e_ab.txt 2>&1
