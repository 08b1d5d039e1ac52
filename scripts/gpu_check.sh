#!/bin/bash
# One gpurun session: build, GPU parity tests, smoke, bench (N=1), ncu launch list + full
# capture of the top kernels.  Outputs under gpurun_out/.
set -u
OUT=gpurun_out
mkdir -p $OUT
TAG=${TAG:-r1}
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { tail -30 $OUT/build_$TAG.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > $OUT/gpu_$TAG.txt
if [ "${TESTS:-1}" = 1 ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q --timeout 600 ${PYTEST_ARGS:-} > $OUT/pytest_gpu_$TAG.log 2>&1
  echo "pytest rc=$?"; tail -5 $OUT/pytest_gpu_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke_$TAG.log
fi
for CFG in ${CONFIGS:-c2}; do
  timeout 600 python bench.py --config $CFG ${BENCH_ARGS:-} > $OUT/bench_${CFG}_$TAG.json 2> $OUT/bench_${CFG}_$TAG.err
  echo "bench $CFG rc=$?"; tail -c 3000 $OUT/bench_${CFG}_$TAG.json; tail -3 $OUT/bench_${CFG}_$TAG.err
done
if [ "${NCU:-1}" = 1 ]; then
  for CFG in ${NCU_CONFIGS:-c2}; do
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'score|select|attn|meta|decode' -c 60 --csv \
      --log-file $OUT/launches_${CFG}_$TAG.csv python bench.py --config $CFG --steps 20 --warmup 3 --no-oracle --no-e2e > /dev/null 2>&1
    echo "ncu launches $CFG rc=$?"
    timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'decode_cluster|sparse_attn' -s 6 -c 3 \
      -o $OUT/prof_${CFG}_$TAG -f python bench.py --config $CFG --steps 10 --warmup 3 --no-oracle --no-e2e > $OUT/ncu_full_${CFG}_$TAG.log 2>&1
    echo "ncu full $CFG rc=$?"; tail -3 $OUT/ncu_full_${CFG}_$TAG.log
  done
fi
