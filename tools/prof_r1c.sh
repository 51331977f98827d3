# round-1c ncu evidence: launch lists (host loop: ncu skips conditional-graph kernels) and
# full-set captures of the dominant kernels of C4 (2D Poisson) and CD2 (complex diffusion)
set -x
python bench.py --config C4 --steps 2 --warmup 3 --no-cpu --no-e2e --host-loop > gpurun_out/r1c_c4_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r1c_C4_launches.csv \
    python bench.py --config C4 --steps 2 --warmup 3 --no-cpu --no-e2e --host-loop > gpurun_out/r1c_c4_ncu.log 2>&1
python bench.py --config CD2-f32 --steps 2 --warmup 3 --no-cpu --no-e2e --host-loop > gpurun_out/r1c_cd2_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r1c_CD2_launches.csv \
    python bench.py --config CD2-f32 --steps 2 --warmup 3 --no-cpu --no-e2e --host-loop > gpurun_out/r1c_cd2_ncu.log 2>&1
python tools/prof_cycle.py C4 2 && ncu --set full --clock-control none --import-source on \
    -k regex:"k_jacobi2d|k_resid_restrict2d|k_prolong2d" --launch-skip 0 --launch-count 3 \
    -o gpurun_out/r1c_C4_full python tools/prof_cycle.py C4 1 > gpurun_out/r1c_c4_full.log 2>&1
python tools/prof_cd.py CD2-f32 2 && ncu --set full --clock-control none --import-source on \
    -k regex:"k_cd_jacobi|k_cd_fas_rhs|k_cd_norm" --launch-skip 0 --launch-count 3 \
    -o gpurun_out/r1c_CD2_full python tools/prof_cd.py CD2-f32 1 > gpurun_out/r1c_cd2_full.log 2>&1
ls -la gpurun_out/ | grep r1c
