#!/bin/bash
# Constant tables built on the host: parity (parity core + 4-bit + wide + faults), A/B timing vs FIX.
set -u
mkdir -p gpurun_out
#timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_4bit.py tests/test_gpu_wide.py tests/test_gpu_fragment.py -q -x > gpurun_out/pytest_const.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pytest_const.log
for v in FIX CONST FIX CONST; do
  echo "== $v"; LTL_LIB=build/ab/$v.so timeout 300 python tools/pk_time2.py 32768
done
