# ncu of the large-batch update GEMM (F2) at m = 8192: launch list of one step, then the source view of one F2
mkdir -p gpurun_out/nl
R=gpurun_out/nl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $R/launches.csv python scripts/bench_config5.py --m-per-gpu 8192 --steps 1 --warmup 1 > $R/l.log 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.DictReader(open('gpurun_out/nl/launches.csv')) if r.get('Metric Name')=='gpu__time_duration.sum']
for i,r in enumerate(rows[:80]):
    print(i, r['Kernel Name'][:60], r['Grid Size'], r['Metric Value'])
PY
