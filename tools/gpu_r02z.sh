#!/bin/bash
# 4-bit cells v2 (bias MMA, 2R): staging-slot / box-stage A/B, ncu.
set -u
mkdir -p gpurun_out
for v in base S4 S4X8 base S4 S4X8; do
  if [[ $v == base ]]; then unset LTL_LIB; else export LTL_LIB=build/ab/$v.so; fi
  echo "== $v"; timeout 300 python tools/pk_time.py 16384 cat-u8 cat; timeout 300 python tools/pk_time.py 32768 cat
done
unset LTL_LIB
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ltl_tc_step -s 3 -c 1 \
  -o gpurun_out/prof_pk2_32768 -f python tools/pk_time.py 32768 cat > gpurun_out/ncu_pk2.log 2>&1; echo "ncu rc=$?"
