# A/B of the fused 2D Jacobi passes on C4 (MG_NO_KFUSE=1 disables them) + their parity tests
timeout 900 python -m pytest tests/test_gpu_kfuse.py tests/test_gpu_2d.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
for v in 0 1; do
  if [ $v = 1 ]; then export MG_NO_KFUSE=1; fi
  timeout 300 python bench.py --no-cpu --no-e2e --config C4 --steps 30 > gpurun_out/kf_$v.json 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/kf_$v.json').read().strip().splitlines()[-1]); print('nokfuse=$v', round(d['ms_per_step'],4), [(k['kernel'], round(k['ms_per_step'],4), k['launches_per_step'], round(k['GBps'])) for k in d['kernels']][:8])"
done
