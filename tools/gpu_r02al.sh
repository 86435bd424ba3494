#!/bin/bash
# 16384^2 persistent sweep: chunk length (units) re-tuned on the current kernel.
set -u
for i in 1 2; do
  for u in 8 12 16 24 32 64 128; do echo "== $u"; LTL_SWEEP_UNITS=$u timeout 300 python tools/pk_time.py 16384 cat | tail -1; done
done
