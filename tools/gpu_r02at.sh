#!/bin/bash
# 32768^2 with 4-bit cells: one launch per generation vs the persistent sweep (chunk lengths); u8 per launch for reference.
set -u
for i in 1 2; do
  echo "== u8 / 4-bit per launch"; timeout 300 python tools/pk_time.py 32768 cat cat-4bit
  for u in 16 32 64 128; do echo "== 4-bit sweep $u"; LTL_FORCE_PERSIST=1 LTL_SWEEP_UNITS=$u timeout 300 python tools/pk_time.py 32768 cat-4bit; done
done
