# A/B of programmatic dependent launch for the 3D level kernels (MG_NO_PDL=1 disables it)
for v in 0 1 0 1; do
  if [ $v = 1 ]; then export MG_NO_PDL=1; else unset MG_NO_PDL; fi
  timeout 300 python bench.py --no-cpu --no-e2e --config C3-f64 --steps 50 > gpurun_out/pdl_$v.json 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/pdl_$v.json').read().strip().splitlines()[-1]); print('nopdl=$v', round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
