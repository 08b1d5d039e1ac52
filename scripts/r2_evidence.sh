#!/bin/bash
# Round-2 evidence run (one gpurun session): build, GPU parity suite, smoke, bench lines for
# every BASELINE workload (+ per-GPU slices, FP8 KV, reference arm), the NEXT-4 sweep, ncu
# launch list + --set full captures of decode_cluster_kernel, phase stamps.  -> gpurun_out/
set -u
OUT=gpurun_out; TAG=${TAG:-r2}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/ev_build.log 2>&1 || { tail -30 $OUT/ev_build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > $OUT/ev_gpu_$TAG.txt
if [ "${TESTS:-1}" = 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -q > $OUT/ev_pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/ev_pytest_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/ev_smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/ev_smoke_$TAG.log
fi
b() {  # tag, args...
  local t=$1; shift
  timeout 900 python bench.py "$@" > $OUT/ev_bench_${t}_$TAG.json 2> $OUT/ev_bench_${t}_$TAG.err
  python - "$OUT/ev_bench_${t}_$TAG.json" "$t" <<'PY'
import json, sys
try:
    j = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = j.get("roofline") or {}
    e = j.get("e2e") or {}
    print(sys.argv[2], "us/step", round(j["ms_per_step"] * 1e3, 2), "value", round(j["value"]), "frac", r.get("frac") and round(r["frac"], 3),
          "e2e", e.get("value") and round(e["value"]), "cpu", (j.get("cpu_baseline") or {}).get("value"), "clk", (j.get("clocks") or {}).get("sm_mhz"))
except Exception as ex:
    print(sys.argv[2], "FAILED", ex)
PY
}
if [ "${BENCH:-1}" = 1 ]; then
  b c2 ; b c3 --config c3 ; b c4 --config c4 ; b c5 --config c5
  b c4-slice8 --config c4 --slice 8 ; b c5-b1 --config c5 --batch 1 ; b c5-slice8 --config c5 --slice 8
  b c5-b1-slice8 --config c5 --batch 1 --slice 8
  b c2-fp8 --config c2 --kv fp8 ; b c3-fp8 --config c3 --kv fp8 ; b c5-fp8 --config c5 --kv fp8 ; b c4-slice8-fp8 --config c4 --slice 8 --kv fp8
  timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/ev_ref_c2_$TAG.json 2>&1; echo "reference rc=$?"; tail -c 400 $OUT/ev_ref_c2_$TAG.json
fi
if [ "${SWEEP:-1}" = 1 ]; then
  timeout 1500 python bench.py --config c3 --sweep > $OUT/ev_sweep_c3_$TAG.json 2> $OUT/ev_sweep_c3_$TAG.err; echo "sweep rc=$?"
fi
if [ "${NCU:-1}" = 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'score|select|attn|meta|decode|quantize' -c 80 --csv \
    --log-file $OUT/ev_launches_c2_$TAG.csv python bench.py --config c2 --steps 20 --warmup 3 --no-oracle --no-e2e --no-reuse --no-spread --no-dense > /dev/null 2>&1
  echo "ncu launches rc=$?"
  n() {  # tag, args...
    local t=$1; shift
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_cluster -s 4 -c 1 \
      -o $OUT/ev_prof_${t}_$TAG -f python scripts/one_step.py "$@" 6 > $OUT/ev_ncu_${t}_$TAG.log 2>&1
    echo "ncu full $t rc=$?"
  }
  n c2 c2 bf16; n c3 c3 bf16; n c5 c5 bf16; n c2-fp8 c2 fp8; n c3-fp8 c3 fp8
  # summaries + DRAM traffic on the box; the reports stay under /tmp (gpurun_out/ is capped at
  # 64 MiB), except the C2 one when it is small
  args=""
  for t in c2 c3 c5 c2-fp8 c3-fp8; do
    r=$OUT/ev_prof_${t}_$TAG.ncu-rep
    [ -f $r ] || continue
    python scripts/ncu_summary.py $r > $OUT/ev_ncusum_${t}_$TAG.txt 2>&1
    ncu -i $r --page raw --csv > $OUT/ev_ncuraw_${t}_$TAG.csv 2>/dev/null
    args="$args $t=$r"
  done
  python scripts/traffic_json.py $args -o $OUT/ev_traffic_$TAG.json > /dev/null 2>&1
  mkdir -p /tmp/ncu_reps; for r in $OUT/ev_prof_*_$TAG.ncu-rep; do
    case $r in *prof_c2_*) [ $(stat -c %s $r) -lt 25000000 ] && continue;; esac
    mv $r /tmp/ncu_reps/
  done
fi
if [ "${STAMPS:-1}" = 1 ]; then
  for c in c2 c3 c5; do timeout 120 python scripts/step_stamps.py $c bf16; done > $OUT/ev_stamps_$TAG.txt 2>&1
  for c in c2 c3; do timeout 120 python scripts/step_stamps.py $c fp8; done >> $OUT/ev_stamps_$TAG.txt 2>&1
fi
exit 0
