#!/bin/bash
# Same-box A/B of the u8 step: the commit before the 4-bit work (OLD) vs now (NEW).
set -u
for v in OLD NEW OLD NEW OLD NEW; do
  echo "== $v"; LTL_LIB=build/ab/$v.so timeout 300 python tools/pk_time.py 32768 cat; LTL_LIB=build/ab/$v.so timeout 300 python tools/pk_time.py 16384 cat
done
