#!/bin/bash
# Development loop on the GPU box: build, GPU parity tests, per-call timings and pipeline
# timelines.  usage: TAG=x CFGS="c2 c3" bash scripts/dev_loop.sh
set -u
OUT=gpurun_out; mkdir -p $OUT; TAG=${TAG:-dev}
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { tail -30 $OUT/build_$TAG.log; exit 1; }
if [ "${TESTS:-1}" = 1 ]; then
  timeout ${TEST_TIMEOUT:-900} python -m pytest tests -m gpu -x -q --timeout 300 ${PYTEST_ARGS:-} > $OUT/pytest_$TAG.log 2>&1
  echo "pytest rc=$?"; tail -4 $OUT/pytest_$TAG.log
fi
for c in ${CFGS:-c2 c3}; do
  timeout 300 python scripts/kbench.py $c 200 2>&1 | tee $OUT/kb_${c}_$TAG.txt
  timeout 300 python scripts/step_stamps.py $c > $OUT/ts_${c}_$TAG.txt 2>&1; head -11 $OUT/ts_${c}_$TAG.txt
done
