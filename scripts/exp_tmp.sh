set -u
python -m paper_2509_12211_b200._build --force > /dev/null 2>&1 || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "s4 or s8" 2>&1 | tail -3
timeout 1500 python bench.py --config c3 --sweep --sweep-S 16,64 --sweep-ratios 0.1,0.3 > gpurun_out/sweep_t.json 2> gpurun_out/sweep_t.err; tail -6 gpurun_out/sweep_t.err
timeout 1500 python bench.py --config c3 --sweep --sweep-S 16 --sweep-ratios 0.1,0.3 --sweep-hot 4,1.0 > gpurun_out/sweep_t.json 2> gpurun_out/sweep_t.err; tail -3 gpurun_out/sweep_t.err
