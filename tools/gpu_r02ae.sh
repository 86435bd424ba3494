#!/bin/bash
# Same-box A/B of the u8 step at 32768^2: OLD (pre-4-bit commit), NEW (now),
# HYB (now, with the pre-4-bit ltl_tc.cu).
set -u
for v in OLD FIX NEW OLD FIX NEW; do
  echo "== $v"; LTL_LIB=build/ab/$v.so timeout 300 python tools/pk_time.py 32768 cat
done
