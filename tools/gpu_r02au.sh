#!/bin/bash
# Dynamic remainder schedule (DYN) vs the static one (STAT): parity, then same-box timing.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ring.py tests/test_gpu_4bit.py -q -x > gpurun_out/pytest_dyn.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pytest_dyn.log
for v in STAT DYN STAT DYN; do
  echo "== $v"
  LTL_LIB=build/ab/$v.so timeout 300 python tools/pk_time.py 32768 cat
  LTL_NO_PERSIST=1 LTL_LIB=build/ab/$v.so timeout 300 python tools/pk_time.py 16384 cat
  LTL_LIB=build/ab/$v.so timeout 300 python tools/pk_time.py 8192 cat
done
for v in STAT DYN; do echo "== $v 65536"; LTL_LIB=build/ab/$v.so timeout 300 python tools/pk_time.py 65536 cat; done
