# A/B of the shared-memory coarse tail (k_tail_sm) against the global-memory one (MG_TAIL_GLOBAL=1)
for v in 0 1; do
  if [ $v = 1 ]; then export MG_TAIL_GLOBAL=1; fi
  for c in C1 C2 C4 C3-f64; do
    timeout 300 python bench.py --no-cpu --no-e2e --config $c --steps 30 > gpurun_out/tail_${c}_$v.json 2>&1
    python -c "
import json
d=json.loads(open('gpurun_out/tail_${c}_$v.json').read().strip().splitlines()[-1]); t=[k for k in d['kernels'] if k['kernel'].startswith('coarse_tail')]
print('$c global=$v', round(d['ms_per_step'],4), [(k['kernel'], round(k['ms_per_step'],4)) for k in t])"
  done
done
