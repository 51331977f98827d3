for mr in 16 8 4; do for tm in 49152 300000; do
MG_PM2_MINROWS=$mr MG_TAIL_MAX=$tm timeout 300 python bench.py --no-cpu --no-e2e --config C4 --steps 30 > gpurun_out/c4_${mr}_${tm}.json 2>&1
python -c "
import json,sys
d=json.loads(open('gpurun_out/c4_${mr}_${tm}.json').read().strip().splitlines()[-1]); print('minrows=$mr tail=$tm', round(d['ms_per_step'],4))"
done; done
