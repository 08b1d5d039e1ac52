python -m paper_2509_12211_b200._build --force > /dev/null 2>&1 || exit 1
for c in ${CONFIGS:-c2 c3 c5}; do
  for ns in ${NS_LIST:-0 1500 2500 3500 5000}; do
    TS_PIPE=0 TS_SC_STAGGER_NS=$ns timeout 120 python bench.py --config $c --steps 200 --warmup 10 --no-oracle --no-dense --no-e2e --no-spread > /tmp/o.json 2>/dev/null
    python -c "import json; j=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); print('$c stagger $ns us/step', round(j['ms_per_step']*1e3,2), 'serial', round(j['serialised_step_us'],2))"
  done
done
