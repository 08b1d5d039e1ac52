set -u
python -m paper_2509_12211_b200._build --force > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp8.py -m gpu -q -x -k "decode_step or fp8" 2>&1 | tail -2
for kv in bf16 fp8; do for c in c2 c3 c5; do timeout 300 python bench.py --config $c --kv $kv --steps 1000 --warmup 10 --no-dense --no-e2e --no-reuse --no-oracle --no-spread 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c $kv us', round(j['ms_per_step']*1e3,2))"; done; done
git stash -q 2>/dev/null; python -m paper_2509_12211_b200._build --force > /dev/null 2>&1
for kv in bf16 fp8; do for c in c2 c3 c5; do timeout 300 python bench.py --config $c --kv $kv --steps 1000 --warmup 10 --no-dense --no-e2e --no-reuse --no-oracle --no-spread 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('BASE $c $kv us', round(j['ms_per_step']*1e3,2))"; done; done
