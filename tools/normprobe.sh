# A/B timing probe for DESIGN §12 lead 4: how much of the C3 sweep+norm head is the black
# nodes' residual stencil. B = the library built with -DMG_PROBE_RED_ONLY_NORM (norm over red
# nodes only: NOT a parity build), A = the default build. Three alternating runs each.
run() { timeout 300 python bench.py --no-cpu --no-e2e --config $1 --steps 50 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$2 $1', round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for i in 1 2 3; do
  make -s -j16 -B lib > /dev/null 2>&1 && run C3-f64 A && run C3-f32 A
  make -s -j16 -B lib MG_EXTRA=-DMG_PROBE_RED_ONLY_NORM > /dev/null 2>&1 && run C3-f64 B && run C3-f32 B
done
make -s -j16 -B lib > /dev/null 2>&1
