# coarse tail: small levels on CTA 0 alone (default, MG_TAIL_SOLO=2048 interior nodes) vs cluster for all (MG_TAIL_SOLO=0)
for v in ${SOLO_LIST:-2048 0}; do
  export MG_TAIL_SOLO=$v
  for c in C1 C2 C4 C3-f64; do
    timeout 300 python bench.py --no-cpu --no-e2e --config $c --steps 30 > gpurun_out/solo_${c}_$v.json 2>&1
    python -c "
import json
d=json.loads(open('gpurun_out/solo_${c}_$v.json').read().strip().splitlines()[-1]); t=[k for k in d['kernels'] if k['kernel'].startswith('coarse_tail')]
print('$c solo=$v', round(d['ms_per_step'],4), [(k['kernel'], round(k['ms_per_step'],4)) for k in t])"
  done
done
