#!/bin/bash
# bench one config under several env settings (development tool; the A/B knobs exist in the
# dev build only, libtinyserve_dev.so, loaded with TS_DEV_LIB=1).
# Usage: CFG=c5 bash scripts/envsweep.sh "TS_SC_TRIGGER=1" "TS_SC_CMAX=8" ...
set -u
python -m paper_2509_12211_b200._build --dev > /dev/null 2>&1
for e in "" "$@"; do
  r=$(env TS_DEV_LIB=1 $e timeout -s KILL 300 python bench.py --config ${CFG:-c5} --no-oracle --no-dense --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value']), round(j['ms_per_step']*1e3,2))")
  echo "${CFG:-c5} [$e] $r"
done
