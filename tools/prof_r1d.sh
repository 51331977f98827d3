# round-1d ncu evidence for the bench line (C3 FP64): launch list of the same bench command
# (host loop: ncu skips kernels of conditional graphs) and a full-set capture of the level-0
# RBGS sweep, the sweep+norm head, the fused residual+restriction and the prolongation
set -x
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --host-loop > gpurun_out/r1d_c3_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1d_C3-f64_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --host-loop > gpurun_out/r1d_c3_ncu.log 2>&1
python tools/prof_cycle.py C3-f64 2 && ncu --set full --clock-control none --import-source on \
    -k regex:"k_sweep3d|k_resid_restrict3d|k_prolong3d" --launch-skip 0 --launch-count 4 \
    -o gpurun_out/r1d_C3-f64_full python tools/prof_cycle.py C3-f64 1 > gpurun_out/r1d_c3_full.log 2>&1
ls -la gpurun_out/ | grep r1d
