set -x
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r1f_gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r1f_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r1f_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r1f_smoke.log
timeout 300 python bench.py > gpurun_out/r1f_bench_default.json 2> gpurun_out/r1f_bench_default.err; echo "bench rc=$?"; tail -1 gpurun_out/r1f_bench_default.json | cut -c1-400
bash tools/bench_all.sh > gpurun_out/r1f_bench_all.log 2>&1; cat gpurun_out/r1f_bench_all.log
bash tools/prof_r1f.sh > gpurun_out/r1f_prof.log 2>&1; tail -5 gpurun_out/r1f_prof.log
