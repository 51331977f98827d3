# complex-diffusion bench lines (kernel breakdown printed compactly)
for c in CD2-f32 CD2-gs-f32 CD2-f64 CD3-f32 CD3-gs-f32; do
  timeout 300 python bench.py --no-cpu --config $c --steps 20 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python - <<PY
import json
d=json.loads(open("gpurun_out/bench_$c.json").read().strip().splitlines()[-1])
print("$c", round(d["ms_per_step"],4), "%.3e" % d["value"], "model GB/s", round(d["model_GBps"]), "frac", round(d["roofline"]["frac"],3), d["roofline"]["kernel"], "e2e", d["e2e"] and round(d["e2e"]["ms_per_step"],2))
for k in d["kernels"][:6]: print("   ", k["kernel"], round(k["ms_per_step"],4), k["launches_per_step"], round(k["GBps"] or 0))
PY
done
