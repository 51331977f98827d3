# round-1e ncu evidence for the bench line (C3 FP64) after the deeper ring prefetch: launch
# list of the same bench command (host loop) and a full-set capture of the L0 RBGS sweep,
# the sweep+norm head and the residual+restriction
set -x
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --host-loop > gpurun_out/r1e_c3_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1e_C3-f64_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --host-loop > gpurun_out/r1e_c3_ncu.log 2>&1
python tools/prof_solve.py C3-f64 1 && ncu --set full --clock-control none --import-source on \
    -k regex:"k_sweep3d|k_resid_restrict3d" --launch-skip 0 --launch-count 3 \
    -o gpurun_out/r1e_C3-f64_full python tools/prof_solve.py C3-f64 1 > gpurun_out/r1e_c3_full.log 2>&1
ls -la gpurun_out/ | grep r1e_C3
