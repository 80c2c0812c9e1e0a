mkdir -p gpurun_out/it
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/it/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/it/pytest_gpu.log
tail -n 2 gpurun_out/it/pytest_gpu.log
timeout 300 python bench.py --steps 200 > gpurun_out/it/bench.log 2>&1; tail -n 1 gpurun_out/it/bench.log
timeout 300 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/it/bench_ref.log 2>&1; tail -n 1 gpurun_out/it/bench_ref.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/it/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/it/b_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep2 -s 20 -c 1 -o gpurun_out/it/sweep2_full python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/it/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:build2 -s 20 -c 1 -o gpurun_out/it/build2_full python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/it/ncu_full_b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dv2 -s 20 -c 1 -o gpurun_out/it/dv2_full python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/it/ncu_full_d.log 2>&1
ls gpurun_out/it
