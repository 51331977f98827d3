# C3 FP64 + FP32 bench lines (kernel breakdown), for A/B of sweep-kernel changes
for c in C3-f64 C3-f32; do
  timeout 300 python bench.py --no-cpu --no-e2e --config $c --steps 30 > gpurun_out/c3ab_$c.json 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/c3ab_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), d['clocks']['reasons'], [(k['kernel'], round(k['ms_per_step'],4), k['launches_per_step'], round(k['GBps'] or 0)) for k in d['kernels']][:5])"
done
