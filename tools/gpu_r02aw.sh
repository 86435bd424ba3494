#!/bin/bash
# Dynamic remainder with the next grab prefetched and the exit ticket only when used (DYN3) vs static (STAT).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ring.py -q -x > gpurun_out/pytest_dyn3.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pytest_dyn3.log
for v in STAT DYN3 STAT DYN3; do
  echo "== $v"
  LTL_LIB=build/ab/$v.so timeout 300 python tools/pk_time.py 32768 cat cat-4bit
  LTL_LIB=build/ab/$v.so timeout 300 python tools/pk_time.py 8192 cat
  LTL_LIB=build/ab/$v.so timeout 300 python tools/pk_time.py 16384 cat
done
