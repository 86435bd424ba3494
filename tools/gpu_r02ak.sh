#!/bin/bash
# Prologue with the band tiles and the A table built concurrently (OVL) vs before (BASE2).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "criterion1 or fault or determinism or persistent" > gpurun_out/pytest_ovl.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pytest_ovl.log
for v in BASE2 OVL BASE2 OVL; do
  echo "== $v"; for n in 32768 16384 8192; do LTL_LIB=build/ab/$v.so timeout 300 python tools/pk_time2.py $n; done
done
