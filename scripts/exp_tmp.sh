set -u
python -m paper_2509_12211_b200._build --force > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "shard" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_nccl.py tests/test_boundary.py -q -x 2>&1 | tail -2
for a in "--slice 8" "--batch 1 --slice 8" "--slice 2"; do timeout 300 python bench.py --config c5 $a --steps 200 --warmup 10 --no-dense --no-e2e --no-reuse --no-oracle --no-spread 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5 $a us', round(j['ms_per_step']*1e3,2), 'launches', j['gpu_launches']/j['steps'])"; done
