mkdir -p gpurun_out/nd
R=gpurun_out/nd
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dv2 -s 3 -c 1 -o $R/dv2 python scripts/step_env.py base > $R/ncu.log 2>&1
ncu -i $R/dv2.ncu-rep --page source --csv --print-source cuda,sass > $R/src.csv 2>/dev/null
python scripts/ncu_lines.py $R/src.csv 40 > $R/lines.txt
python scripts/ncu_summary.py full $R/dv2.ncu-rep > $R/summary.txt 2>&1
head -32 $R/summary.txt; cat $R/lines.txt
