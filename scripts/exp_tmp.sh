set -u
bash scripts/r2_fp8.sh
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
for c in c2 c3 c5; do for kv in bf16 fp8; do timeout 300 python bench.py --config $c --kv $kv --steps 200 --warmup 10 --no-dense --no-e2e --no-reuse --no-oracle --no-spread 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c $kv us', round(j['ms_per_step']*1e3,2), 'frac', round(j['roofline']['frac'],3))"; done; done
for kv in bf16 fp8; do timeout 120 python scripts/step_stamps.py c2 $kv | grep -E "selected|consumed|end"; done
