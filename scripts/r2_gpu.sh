# Round-2 GPU loop: build, GPU parity tests (optionally filtered), bench lines (20-step driver
# protocol) for the given configs.  usage: TAG=x CONFIGS="c2 c3" PYTEST_K="..." bash scripts/r2_gpu.sh
set -u
mkdir -p gpurun_out
TAG=${TAG:-dev}
python -m paper_2509_12211_b200._build --force > gpurun_out/${TAG}_build.log 2>&1 || { tail -20 gpurun_out/${TAG}_build.log; exit 1; }
if [ "${TESTS:-1}" = 1 ]; then
  timeout -s KILL 1200 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/${TAG}_pytest.log | grep -v "^\s*$" | tail -8
fi
for c in ${CONFIGS:-c2}; do
  timeout -s KILL 300 python bench.py --config $c --steps ${STEPS:-20} --warmup ${WARMUP:-5} ${BENCH_ARGS:---no-oracle --no-dense --no-e2e --no-reuse} > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  python - "$c" "$TAG" <<'PY'
import json, sys
c, tag = sys.argv[1], sys.argv[2]
try:
    j = json.loads(open(f"gpurun_out/{tag}_bench_{c}.json").read().strip().splitlines()[-1])
    sp = j.get("spread") or {}
    print(c, "us/step", round(j["ms_per_step"] * 1e3, 2), "frac", round(j["roofline"]["frac"], 3),
          "serial", j.get("serialised_step_us") and round(j["serialised_step_us"], 2),
          "p10/50/90", [round(sp.get(k, 0), 2) for k in ("us_per_step_p10", "us_per_step_median", "us_per_step_p90")],
          "warmL2", sp.get("warm_l2_us_per_step") and round(sp["warm_l2_us_per_step"], 2),
          "readpk", (j.get("read_peak") or {}).get("gbs"), "clk", j["clocks"]["sm_mhz"])
    ru = j.get("reuse") or {}
    if ru: print("   reuse", {k: (round(v, 3) if isinstance(v, float) else v) for k, v in ru.items() if k not in ("workload", "api")})
except Exception as ex:
    print(c, "bench failed", ex); print(open(f"gpurun_out/{tag}_bench_{c}.err").read()[-2500:])
PY
done
