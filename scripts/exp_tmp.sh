set -u
python -m paper_2509_12211_b200._build --force > /dev/null 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for c in c2 c3 c5; do for kv in bf16 fp8; do timeout 300 python bench.py --config $c --kv $kv --steps 200 --warmup 10 --no-dense --no-e2e --no-reuse --no-oracle --no-spread 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c $kv us', round(j['ms_per_step']*1e3,2), 'frac', round(j['roofline']['frac'],3))"; done; done
