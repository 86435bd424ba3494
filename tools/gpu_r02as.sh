#!/bin/bash
# Warp-uniform TMEM addresses (SHFL: no per-use R2UR in the convert / output loops) vs before (BASE3).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_4bit.py -q -x -k "criterion1 or fault or determinism or oracle or persistent" > gpurun_out/pytest_shfl.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pytest_shfl.log
for v in BASE3 SHFL BASE3 SHFL; do
  echo "== $v"; LTL_LIB=build/ab/$v.so timeout 300 python tools/pk_time.py 32768 cat cat-4bit; LTL_LIB=build/ab/$v.so timeout 300 python tools/pk_time.py 16384 cat cat-4bit
done
