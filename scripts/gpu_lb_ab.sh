mkdir -p gpurun_out/lbab
for f in 0 1; do
FASTH_LB_DERIVED=$f timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lbab/l$f.csv python scripts/bench_config5.py --m-per-gpu 8192 --steps 1 --warmup 1 > /dev/null 2>&1
done
