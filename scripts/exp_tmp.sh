set -u
python -m paper_2509_12211_b200._build > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "append" 2>&1 | tail -1
for c in c2 c3 c5; do timeout 300 python scripts/app_vs_plain.py $c; done
