#!/bin/bash
# compute-sanitizer over the decode-step parity tests (release + FP8), all four tools.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
K1="test_decode_step and (c3_small or g4_s32 or two_level or g8_s4 or c2_small or c1_ragged)"
K2="test_decode_step_fp8 and (c3_small or two_level) or test_kv_quantize_edge or test_meta_append_fp8"
for tool in memcheck racecheck synccheck initcheck; do
  timeout -s KILL 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "$K1" > gpurun_out/san_${tool}.log 2>&1
  echo "$tool bf16 rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/san_${tool}.log | tail -2 | tr '\n' ' ')"
  timeout -s KILL 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_fp8.py -m gpu -q -x -p no:cacheprovider -k "$K2" > gpurun_out/san_${tool}_fp8.log 2>&1
  echo "$tool fp8 rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/san_${tool}_fp8.log | tail -2 | tr '\n' ' ')"
done
