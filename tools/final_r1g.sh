set -x
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r1g_gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r1g_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r1g_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r1g_smoke.log
timeout 300 python bench.py > gpurun_out/r1g_bench_default.json 2> gpurun_out/r1g_bench_default.err; echo "bench rc=$?"; tail -1 gpurun_out/r1g_bench_default.json | cut -c1-600
