# round-1f ncu evidence for the bench line (C3 FP64) after the flat prolongation (and the
# shared-memory changes measured by tools/eshab.sh): launch list of the same bench command
# (host loop) and a full-set capture of the L0 sweep, sweep+norm head, residual+restriction
# and prolongation
set -x
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --host-loop > gpurun_out/r1f_c3_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1f_C3-f64_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --host-loop > gpurun_out/r1f_c3_ncu.log 2>&1
python tools/prof_solve.py C3-f64 1 && ncu --set full --clock-control none --import-source on \
    -k regex:"k_sweep3d|k_resid_restrict3d|k_prolong3d" --launch-skip 0 --launch-count 30 \
    -o gpurun_out/r1f_C3-f64_full python tools/prof_solve.py C3-f64 1 > gpurun_out/r1f_c3_full.log 2>&1
python tools/prof_solve.py C3-f32 1 && ncu --set full --clock-control none --import-source on \
    -k regex:"k_sweep3d|k_resid_restrict3d|k_prolong3d" --launch-skip 0 --launch-count 30 \
    -o gpurun_out/r1f_C3-f32_full python tools/prof_solve.py C3-f32 1 > gpurun_out/r1f_c3f32_full.log 2>&1
ls -la gpurun_out/ | grep r1f_
