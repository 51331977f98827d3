set -x
bash tools/bench_all_r1g.sh > gpurun_out/r1g_bench_all.log 2>&1; cat gpurun_out/r1g_bench_all.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r1g_C3-f64_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r1g_c3_ncu.log 2>&1; echo "ncu rc=$?"
