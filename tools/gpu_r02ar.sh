#!/bin/bash
# 4-bit cells: bias by a 7th pass-1 MMA (PKB1) vs add.f16x2 in the convert (PKB0); u8 for reference.
set -u
for v in PKB1 PKB0 PKB1 PKB0; do
  echo "== $v"; LTL_LIB=build/ab/$v.so timeout 300 python tools/pk_time.py 32768 cat cat-4bit; LTL_LIB=build/ab/$v.so timeout 300 python tools/pk_time.py 16384 cat-4bit
done
LTL_LIB=build/ab/PKB0.so timeout 600 python tools/pk_check.py 2>&1 | grep -i 'mismatch\|fault' | tail -5
