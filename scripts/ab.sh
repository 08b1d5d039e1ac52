#!/bin/bash
# A/B the in-tree libtinyserve.so against ab/libprev.so on the same box (development tool).
# Usage: CONFIGS="c3 c5" ROUNDS=2 bash scripts/ab.sh
set -u
python -m paper_2509_12211_b200._build > /dev/null 2>&1
cp paper_2509_12211_b200/libtinyserve.so ab/libcur.so
for r in $(seq 1 ${ROUNDS:-2}); do
  for v in cur prev; do
    cp ab/lib$v.so paper_2509_12211_b200/libtinyserve.so
    for c in ${CONFIGS:-c3 c5}; do
      timeout -s KILL 300 python bench.py --config $c --no-oracle --no-dense --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$v', '$c', round(j['value']), round(j['ms_per_step']*1e3,2))"
    done
  done
done
cp ab/libcur.so paper_2509_12211_b200/libtinyserve.so
