# ncu full capture of the fused 2D Jacobi passes (k_jacobi2d_k) on C4, level 0 first
set -x
python tools/prof_cycle.py C4 2 && ncu --set full --clock-control none --import-source on \
    -k regex:"k_jacobi2d_k" --launch-skip 0 --launch-count 2 \
    -o gpurun_out/r1e_C4_kf_full python tools/prof_cycle.py C4 1 > gpurun_out/r1e_c4_kf.log 2>&1
ls -la gpurun_out/ | grep r1e
