# round-1e ncu evidence for C4 after temporal blocking: the bench line, the launch list of the
# same command (host loop), and full-set captures of the fused passes + residual/restriction
set -x
python bench.py --config C4 --steps 20 --warmup 5 --no-cpu > gpurun_out/r1e_c4_bench.json 2>&1
python bench.py --config C4 --steps 2 --warmup 3 --no-cpu --no-e2e --host-loop > gpurun_out/r1e_c4_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r1e_C4_launches.csv \
    python bench.py --config C4 --steps 2 --warmup 3 --no-cpu --no-e2e --host-loop > gpurun_out/r1e_c4_ncu.log 2>&1
python tools/prof_solve.py C4 2 && ncu --set full --clock-control none --import-source on \
    -k regex:"k_jacobi2d_k|k_resid_restrict2d" --launch-skip 0 --launch-count 4 \
    -o gpurun_out/r1e_C4_full python tools/prof_solve.py C4 1 > gpurun_out/r1e_c4_full.log 2>&1
ls -la gpurun_out/ | grep r1e
# the dominant kernel of the C4 step: prolongation fused into the first post pass at L0
# (launch 12 of k_jacobi2d_k in a cycle: head, 5 zero-guess passes L1..L5, CORR L5..L0)
python tools/prof_solve.py C4 1 && ncu --set full --clock-control none --import-source on \
    -k regex:"k_jacobi2d_k" --launch-skip 11 --launch-count 1 \
    -o gpurun_out/r1e_C4_corr_full python tools/prof_solve.py C4 1 > gpurun_out/r1e_c4_corr.log 2>&1
