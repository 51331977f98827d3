# A/B timing: bench lines of C3 with the product lib and experimental libs (MG_LIBRARY)
summ() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['ms_per_step'],4), d['clocks']['sm_mhz'], [(k['kernel'], round(k['ms_per_step'],3)) for k in d['kernels'][:5]])" $1 "$2"; }
for spec in "$@"; do
  lib=${spec%%:*}; rest=${spec#*:}; cfg=${rest%%:*}; flags=${rest#*:}; [ "$flags" = "$rest" ] && flags=""
  L=""; [ "$lib" != "prod" ] && L="MG_LIBRARY=exp/lib_$lib.so"
  env $L python bench.py --config $cfg --no-cpu --no-e2e --no-c5 $flags > gpurun_out/exp_$lib_$cfg.json 2>gpurun_out/exp_err.txt || tail -3 gpurun_out/exp_err.txt
  summ gpurun_out/exp_$lib_$cfg.json "$lib $cfg $flags"
done
