# round-1e ncu evidence for the CD3 plane-marching Jacobi sweep / norm (kernels_cd3d.cu):
# launch list of the bench command (host loop) and a full-set capture of the first launches
set -x
python bench.py --config CD3-f32 --steps 2 --warmup 3 --no-cpu --no-e2e --host-loop > gpurun_out/r1e_cd3_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r1e_CD3_launches.csv \
    python bench.py --config CD3-f32 --steps 2 --warmup 3 --no-cpu --no-e2e --host-loop > gpurun_out/r1e_cd3_ncu.log 2>&1
python tools/prof_cd.py CD3-f32 1 && ncu --set full --clock-control none --import-source on \
    -k regex:"k_cd_jacobi3d|k_cd_gfield_vec" --launch-skip 0 --launch-count 3 \
    -o gpurun_out/r1e_CD3_full python tools/prof_cd.py CD3-f32 1 > gpurun_out/r1e_cd3_full.log 2>&1
ls -la gpurun_out/ | grep r1e_CD3
