set -u
mkdir -p gpurun_out
python -m paper_2509_12211_b200._build --force > gpurun_out/b0_build.log 2>&1 || { tail -20 gpurun_out/b0_build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/b0_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/b0_pytest.log
for c in c2 c3 c5; do
  timeout -s KILL 300 python bench.py --config $c --steps 20 --warmup 5 --no-oracle --no-dense --no-e2e > gpurun_out/b0_${c}_20.json 2>&1
  python -c "import json,sys; j=json.loads(open('gpurun_out/b0_${c}_20.json').read().strip().splitlines()[-1]); print('$c 20steps us', round(j['ms_per_step']*1e3,2), 'serial', round(j['roofline']['phase_us']['serialised_step_us'],2))"
  timeout -s KILL 300 python bench.py --config $c --steps 3000 --warmup 30 --no-oracle --no-dense --no-e2e > gpurun_out/b0_${c}_3000.json 2>&1
  python -c "import json,sys; j=json.loads(open('gpurun_out/b0_${c}_3000.json').read().strip().splitlines()[-1]); print('$c 3000steps us', round(j['ms_per_step']*1e3,2))"
done
