# A/B of the 3D prolongation variants (MG_PROLONG_V, kernels_pm.cu launch_prolong):
# parity of every variant (3D tests that run the prolongation), then the C3 FP64/FP32
# bench lines with the prolongation's per-step time.
set -u
mkdir -p gpurun_out/prolab
# variants (launch_prolong): 0 flat 2 planes/item 6 CTAs (default), 1 marching, 2 marching pipelined,
# 3 flat 8 CTAs (one fine plane per item with 8 / 6 CTAs and two coarse planes per item with
# 4 / 5 CTAs were measured and removed: profiles/r1f/prolab2.txt, prolab3.txt)
for v in 0 1 2 3; do
  MG_PROLONG_V=$v timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_gpu_shapes.py \
      tests/test_gpu_random.py tests/test_gpu_slab_loopback.py \
      > gpurun_out/prolab/t_$v.log 2>&1
  echo "v=$v tests rc=$? $(tail -1 gpurun_out/prolab/t_$v.log)"
done
for rep in 1 2; do
for v in 0 1 2 3; do
  for c in C3-f64 C3-f32; do
    MG_PROLONG_V=$v timeout 300 python bench.py --no-cpu --no-e2e --config $c --steps 30 > gpurun_out/prolab/b_${v}_${c}_$rep.json 2>&1
    python -c "
import json
d=json.loads(open('gpurun_out/prolab/b_${v}_${c}_$rep.json').read().strip().splitlines()[-1])
k=[x for x in d['kernels'] if x['kernel'].startswith('prolong')]
print('v=$v', '$c', round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'], [(x['kernel'], round(x['ms_per_step'],4), round(x['GBps'] or 0)) for x in k])"
  done
done
done
