#!/bin/bash
# 32768^2: one launch per generation vs the persistent sweep with long chunks.
set -u
for i in 1 2; do
  echo "== per launch"; timeout 300 python tools/pk_time.py 32768 cat
  for u in 256 128 64; do
    echo "== sweep, $u-unit chunks"; LTL_FORCE_PERSIST=1 LTL_SWEEP_UNITS=$u timeout 300 python tools/pk_time.py 32768 cat
  done
done
echo "== 65536 per launch"; timeout 300 python tools/pk_time.py 65536 cat
echo "== 65536 sweep 256"; LTL_FORCE_PERSIST=1 LTL_SWEEP_UNITS=256 timeout 300 python tools/pk_time.py 65536 cat
echo "== 65536 sweep 512"; LTL_FORCE_PERSIST=1 LTL_SWEEP_UNITS=512 timeout 300 python tools/pk_time.py 65536 cat
