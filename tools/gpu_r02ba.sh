#!/bin/bash
# Dynamic remainder grab sizes: (min units, fair-share divisor) = (8,2) default, (4,2), (16,2), (8,4).
set -u
for i in 1 2; do for v in D82 D42 D162 D84; do echo "== $v"; LTL_LIB=build/ab/$v.so timeout 300 python tools/pk_time.py 32768 cat | tail -1; LTL_LIB=build/ab/$v.so timeout 300 python tools/pk_time.py 65536 cat | tail -1; done; done
