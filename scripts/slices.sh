python -m paper_2509_12211_b200._build --force > /dev/null 2>&1 || exit 1
run() { tag=$1; shift; timeout 300 python bench.py "$@" --steps 200 --warmup 10 --no-oracle --no-dense --no-e2e --no-reuse > gpurun_out/sl_$tag.json 2> gpurun_out/sl_$tag.err;
  python -c "import json; j=json.loads(open('gpurun_out/sl_$tag.json').read().strip().splitlines()[-1]); print('$tag', 'us/step', round(j['ms_per_step']*1e3,2), 'frac', round(j['roofline']['frac'],3), 'bytes', j['roofline']['algorithmic_bytes_per_launch'], 'R', j['config']['replicas'])" || tail -5 gpurun_out/sl_$tag.err; }
run c4_slice8 --config c4 --slice 8
run c4_full --config c4
run c5_b1 --config c5 --batch 1
run c5_b4 --config c5
run c5_slice8 --config c5 --slice 8
run c5_slice2 --config c5 --slice 2
run c5_b1_slice8 --config c5 --batch 1 --slice 8
