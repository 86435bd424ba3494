#!/bin/bash
# 16384^2 / 8192^2 after the prologue fix: persistent sweep vs one launch per generation.
set -u
for i in 1 2; do
  for n in 16384 8192 4096; do
    echo "== $n sweep (default)"; timeout 300 python tools/pk_time.py $n cat
    echo "== $n per launch"; LTL_NO_PERSIST=1 timeout 300 python tools/pk_time.py $n cat
  done
done
