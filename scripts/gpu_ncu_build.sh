mkdir -p gpurun_out/nb
R=gpurun_out/nb
timeout 600 ncu --set full --clock-control none --import-source on -k regex:build4 -s 3 -c 1 -o $R/build4 python scripts/step_env.py base > $R/ncu.log 2>&1
ncu -i $R/build4.ncu-rep --page source --csv --print-source cuda,sass > $R/src.csv 2>/dev/null
python scripts/ncu_lines.py $R/src.csv 60 > $R/lines.txt
python scripts/ncu_summary.py full $R/build4.ncu-rep > $R/summary.txt 2>&1
head -30 $R/summary.txt; cat $R/lines.txt
