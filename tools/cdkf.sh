# A/B of the fused complex-diffusion Jacobi passes (MG_NO_KFUSE=1 disables them)
for v in 0 1; do
  if [ $v = 1 ]; then export MG_NO_KFUSE=1; fi
  for c in CD2-f32 CD2-f64; do
    timeout 300 python bench.py --no-cpu --no-e2e --config $c --steps 20 > gpurun_out/cdkf_${c}_$v.json 2>&1
    python -c "
import json
d=json.loads(open('gpurun_out/cdkf_${c}_$v.json').read().strip().splitlines()[-1]); print('$c nokfuse=$v', round(d['ms_per_step'],4), [(k['kernel'], round(k['ms_per_step'],4), k['launches_per_step'], round(k['GBps'] or 0)) for k in d['kernels']][:7])"
  done
done
