#!/bin/bash
# Re-entry check: build, full GPU parity suite, smoke, bench lines for c2/c3/c5 + per-GPU slices.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
TAG=${TAG:-chk} CONFIGS="${CONFIGS:-c2 c3 c5}" bash scripts/r2_gpu.sh
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
[ "${SLICES:-1}" = 1 ] && bash scripts/slices.sh
exit 0
