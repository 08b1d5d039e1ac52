#!/bin/bash
# A/B the working tree against ab/prev/ (a checkout of an earlier commit with its own build)
# on the same box (development tool).  Prepare: git worktree add ab/prev <commit>; build there.
# Usage: CONFIGS="c3 c5" ROUNDS=2 bash scripts/ab.sh
set -u
python -m paper_2509_12211_b200._build > /dev/null 2>&1
(cd ab/prev && python -m paper_2509_12211_b200._build > /dev/null 2>&1)
for r in $(seq 1 ${ROUNDS:-2}); do
  for v in cur prev; do
    d=.; [ $v = prev ] && d=ab/prev
    for c in ${CONFIGS:-c3 c5}; do
      (cd $d && timeout -s KILL 300 python bench.py --config $c --no-oracle --no-dense ${AB_ARGS:---no-e2e} 2>/dev/null | tail -1) | python -c "import json,sys; j=json.loads(sys.stdin.read()); e=j.get('e2e') or {}; print('$v', '$c', round(j['value']), round(j['ms_per_step']*1e3,2), 'e2e', e.get('value') and round(e['value']))"
    done
  done
done
