# A/B of two shared-memory-wavefront reductions in the 3D level kernels (kernels_pm.cu):
#   MG_ESH  (bit 0 = FP64, bit 1 = FP32): x-edge values by warp shuffle (sweep, norm, resid+restrict)
#   MG_RRXS (same bits): full-weighting x-sums formed in registers (resid+restrict)
# 3D parity with both on, then C3 FP64/FP32 bench lines for each combination.
set -u
mkdir -p gpurun_out/eshab
for combo in "3 3" "0 3"; do
  set -- $combo
  MG_ESH=$1 MG_RRXS=$2 timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_gpu_shapes.py \
      tests/test_gpu_random.py tests/test_gpu_slab_loopback.py tests/test_gpu_variants.py > gpurun_out/eshab/t_$1_$2.log 2>&1
  echo "ESH=$1 RRXS=$2 tests rc=$? $(tail -1 gpurun_out/eshab/t_$1_$2.log)"
done
for rep in 1 2; do
for combo in "0 0" "3 0" "0 3" "3 3"; do
  set -- $combo
  for c in C3-f64 C3-f32; do
    o=gpurun_out/eshab/b_$1_$2_${c}_$rep.json
    MG_ESH=$1 MG_RRXS=$2 timeout 300 python bench.py --no-cpu --no-e2e --config $c --steps 30 > $o 2>&1
    python -c "
import json
d=json.loads(open('$o').read().strip().splitlines()[-1])
print('esh=$1 xs=$2', '$c', round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'], [(x['kernel'], round(x['ms_per_step'],4), round(x['GBps'] or 0)) for x in d['kernels']][:6])"
  done
done
done
