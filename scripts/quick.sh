#!/bin/bash
# Development loop on the GPU box: rebuild, GPU parity tests, bench summary lines (no oracle /
# dense legs), optional stamp timelines.  Usage: CONFIGS="c2 c3" STAMPS="c3" bash scripts/quick.sh
set -u
mkdir -p gpurun_out
python -m paper_2509_12211_b200._build --force > gpurun_out/q_build.log 2>&1 || { tail -20 gpurun_out/q_build.log; exit 1; }
if [ "${TESTS:-1}" = 1 ]; then
  timeout -s KILL 600 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/q_pytest.log
fi
for c in ${STAMPS:-}; do timeout -s KILL 120 python scripts/step_stamps.py $c; done
for c in ${CONFIGS:-c2 c3 c5}; do
  timeout -s KILL 300 python bench.py --config $c --no-oracle --no-dense ${BENCH_ARGS:-} > gpurun_out/q_bench_$c.json 2> gpurun_out/q_bench_$c.err
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
try:
    j = json.loads(open(f"gpurun_out/q_bench_{c}.json").read().strip().splitlines()[-1])
    e = j.get("e2e") or {}
    print(c, "steps/s", round(j["value"]), "us", round(j["ms_per_step"] * 1e3, 2), "frac", round(j["roofline"]["frac"], 3), "e2e", e.get("value") and round(e["value"]), "clk", j["clocks"]["sm_mhz"])
except Exception as ex:
    print(c, "bench failed", ex); print(open(f"gpurun_out/q_bench_{c}.err").read()[-1500:])
PY
done
