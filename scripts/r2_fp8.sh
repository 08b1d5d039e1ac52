#!/bin/bash
# FP8 KV dev loop: build, FP8 parity tests, bf16 decode-step parity subset (regression).
set -u
mkdir -p gpurun_out
python -m paper_2509_12211_b200._build --force > gpurun_out/f8_build.log 2>&1 || { tail -20 gpurun_out/f8_build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests/test_gpu_fp8.py -m gpu -q -x --durations=8 ${PYTEST_ARGS:-} > gpurun_out/f8_pytest.log 2>&1; echo "fp8 pytest rc=$?"; grep -E "passed|failed|Error|assert|^[0-9.]+s call" gpurun_out/f8_pytest.log | tail -15
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "decode_step" > gpurun_out/f8_reg.log 2>&1; echo "bf16 step rc=$?"; tail -2 gpurun_out/f8_reg.log
exit 0
