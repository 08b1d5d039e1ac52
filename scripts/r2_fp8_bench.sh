#!/bin/bash
# FP8 KV: parity + bench lines (bf16 vs fp8) for c2 / c3 / c5 / c4-slice.
set -u
bash scripts/r2_fp8.sh
for c in c2 c3 c5; do
  for kv in bf16 fp8; do
    timeout -s KILL 300 python bench.py --config $c --kv $kv --steps 200 --warmup 10 --no-dense --no-e2e --no-reuse ${BENCH_ARGS:-} > gpurun_out/f8b_${c}_${kv}.json 2> gpurun_out/f8b_${c}_${kv}.err
    python -c "import json; j=json.loads(open('gpurun_out/f8b_${c}_${kv}.json').read().strip().splitlines()[-1]); r=j['roofline']; print('$c $kv us/step', round(j['ms_per_step']*1e3,2), 'bytes', j['algorithmic_bytes_per_step'], 'frac', round(r['frac'],3), 'cpu', j['cpu_baseline'] and round(j['cpu_baseline']['value'],1))" || tail -5 gpurun_out/f8b_${c}_${kv}.err
  done
done
