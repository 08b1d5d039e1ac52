#!/bin/bash
set -u
mkdir -p gpurun_out
python -m paper_2509_12211_b200._build --force > /dev/null 2>&1 || exit 1
for c in c2 c3; do for kv in bf16 fp8; do timeout 120 python scripts/step_stamps.py $c $kv; done; done
for c in c2; do for kv in bf16 fp8; do
  timeout 300 ncu --set full --clock-control none -k regex:decode_cluster --launch-skip 3 --launch-count 1 -o gpurun_out/f8prof_${c}_${kv} -f python scripts/one_step.py $c $kv 5 > /dev/null 2>&1
  ncu -i gpurun_out/f8prof_${c}_${kv}.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__inst_executed_pipe_tensor_op_hmma.avg.pct_of_peak_sustained_active,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__occupancy_limit_registers,sm__maximum_warps_per_active_cycle_pct,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio 2>/dev/null | tail -1 | cut -c1-600
done; done
