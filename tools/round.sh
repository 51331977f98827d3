#!/bin/bash
# One parameterised GPU measurement script (run on a B200 through gpurun, from the repo root):
#   bash tools/round.sh TAG stage [stage ...]
# stages:
#   tests      pytest -m gpu                              -> gpurun_out/TAG/gpu_tests.log
#   smoke      __graft_entry__.smoke()                    -> gpurun_out/TAG/smoke.log
#   bench      default bench line (C3 FP64)               -> gpurun_out/TAG/bench_default.json
#   benchall   every bench config + the reference arm     -> gpurun_out/TAG/bench/<config>.json
#   launches   ncu launch list of the default bench command (host loop)  -> TAG/C3-f64_launches.csv
#   full:CFG   ncu --set full of CFG's level-0 3D kernels (tools/prof_solve.py) -> TAG/CFG_full.ncu-rep
#   sanitize   compute-sanitizer memcheck/racecheck/synccheck/initcheck over tools/sanitize.py
#   ab:CFG     bench CFG three times (A/B runs of a kernel change)  -> TAG/ab_CFG.txt
#   bmeas:CFG  ncu DRAM bytes of one whole cycle (all kernels)      -> profiles/ncu_cycle_bytes.json
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
summ() {  # one summary line of a bench JSON line
  python - "$1" "$2" <<'PY'
import json, sys
name, path = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(path).read().strip().splitlines()[-1])
except Exception as e:
    print(name, "no line:", e); sys.exit(0)
r = d.get("roofline") or {}
print(name, round(d.get("ms_per_step", 0), 4), "%.3e" % d.get("value", 0), "frac", round(r.get("frac", 0), 3),
      r.get("kernel"), "e2e %.3e" % ((d.get("e2e") or {}).get("value") or 0), (d.get("clocks") or {}).get("sm_mhz"),
      (d.get("clocks") or {}).get("reasons"), d.get("gpu_launches"))
PY
}
for st in "$@"; do
  case $st in
    tests)
      timeout 2400 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests.log 2>&1; echo "pytest rc=$?"
      tail -3 $OUT/gpu_tests.log ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
      tail -2 $OUT/smoke.log ;;
    bench)
      timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; echo "bench rc=$?"
      summ default $OUT/bench_default.json ;;
    benchall)
      mkdir -p $OUT/bench
      for c in C3-f64 C3-f32 C5 C2 C4 C1 C2-lex CD2-f32 CD2-gs-f32 CD2-f64 CD3-f32 CD3-gs-f32; do
        timeout 600 python bench.py --config $c > $OUT/bench/$c.json 2> $OUT/bench/$c.err
        summ $c $OUT/bench/$c.json
      done
      timeout 600 python bench.py --config C4 --no-kfuse --no-cpu --no-e2e > $OUT/bench/C4-nokfuse.json 2> $OUT/bench/C4-nokfuse.err
      summ C4-nokfuse $OUT/bench/C4-nokfuse.json
      timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench/reference_C3-f64.json 2>&1
      tail -1 $OUT/bench/reference_C3-f64.json | cut -c1-300 ;;
    launches)
      python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-c5 --host-loop > $OUT/launches_plain.json 2>&1 && \
      ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/C3-f64_launches.csv \
          python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-c5 --host-loop > $OUT/launches_ncu.log 2>&1
      echo "launches rc=$?"
      python tools/launch_shares.py $OUT/C3-f64_launches.csv > $OUT/C3-f64_launch_shares.txt 2>&1
      head -20 $OUT/C3-f64_launch_shares.txt ;;
    full:*)
      cfg=${st#full:}
      python tools/prof_solve.py $cfg 1 > /dev/null 2>&1 && \
      ncu --set full --clock-control none --import-source on \
          -k regex:"k_sweep3d|k_resid_restrict3d|k_prolong3d" --launch-skip 0 --launch-count 30 \
          -o $OUT/${cfg}_full python tools/prof_solve.py $cfg 1 > $OUT/${cfg}_full.log 2>&1
      echo "full $cfg rc=$?"
      python tools/ncu_summary.py $OUT/${cfg}_full.ncu-rep > $OUT/${cfg}_full_summary.txt 2>&1
      head -40 $OUT/${cfg}_full_summary.txt ;;
    bmeas:*)  # SURVEY §8(d) B_meas: DRAM bytes of one cycle (all kernels) -> profiles/ncu_cycle_bytes.json
      cfg=${st#bmeas:}
      for n in 1 2; do
        ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
            --log-file $OUT/${cfg}_bmeas_$n.csv python tools/prof_solve.py $cfg $n > /dev/null 2>&1
      done
      python tools/ncu_cycle_bytes.py $cfg $OUT/${cfg}_bmeas_1.csv $OUT/${cfg}_bmeas_2.csv ;;
    sanitize)  # compute-sanitizer (closed on this pool) then the checked build
      mkdir -p $OUT/sanitizer
      python tools/sanitize.py > $OUT/sanitizer/plain.log 2>&1; echo "sanitize plain rc=$?"
      MG_LIBRARY=paper_1406_5369_b200/libmgb200_checked.so CUDA_LAUNCH_BLOCKING=1 python tools/sanitize.py \
        > $OUT/sanitizer/checked_build.log 2>&1; echo "checked build rc=$?"; tail -3 $OUT/sanitizer/checked_build.log
      for tool in memcheck initcheck synccheck racecheck; do
        timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
          python tools/sanitize.py > $OUT/sanitizer/$tool.log 2>&1
        echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|error" $OUT/sanitizer/$tool.log | sort | uniq -c | head -8
      done ;;
    ab:*)
      cfg=${st#ab:}
      for i in 1 2 3; do
        timeout 600 python bench.py --config $cfg --no-cpu --no-e2e --no-c5 > $OUT/ab_${cfg}_$i.json 2> /dev/null
        summ "$cfg#$i" $OUT/ab_${cfg}_$i.json
      done | tee $OUT/ab_${cfg}.txt ;;
    *) echo "unknown stage $st" ;;
  esac
done
