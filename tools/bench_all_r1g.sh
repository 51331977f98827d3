# every bench config once (default settings) -> gpurun_out/r1g_bench/<config>.json
mkdir -p gpurun_out/r1g_bench
for c in C3-f64 C3-f32 C5 C2 C4 C1 C2-lex CD2-f32 CD2-gs-f32 CD2-f64 CD3-f32 CD3-gs-f32; do
  timeout 600 python bench.py --config $c > gpurun_out/r1g_bench/$c.json 2> gpurun_out/r1g_bench/$c.err
  python - <<PY
import json
d=json.loads(open("gpurun_out/r1g_bench/$c.json").read().strip().splitlines()[-1])
cpu=d.get("cpu_baseline") or {}
print("$c", round(d["ms_per_step"],4), "%.3e" % d["value"], "frac", round(d["roofline"]["frac"],3), d["roofline"]["kernel"],
      "e2e %.3e" % (d["e2e"] or {}).get("value", 0), "cpu %.3e" % cpu.get("value", 0), cpu.get("cores"), d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d["gpu_launches_per_step"])
PY
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r1g_bench/reference_C3-f64.json 2>&1
tail -1 gpurun_out/r1g_bench/reference_C3-f64.json | cut -c1-300
