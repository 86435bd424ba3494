#!/bin/bash
# 4-bit cells, why slower: per-site waits (trace build) packed vs u8, 8 vs 9
# box stages, ncu of the packed step kernel.
set -u
mkdir -p gpurun_out
for e in 0 1; do
  if [[ $e == 1 ]]; then export LTL_U8_CELLS=1; else unset LTL_U8_CELLS; fi
  echo "== u8=$e"
  LTL_LIB=build/ab/TR.so timeout 300 python tools/trace_waits.py 16384 10
  LTL_NO_PERSIST=1 LTL_LIB=build/ab/TR.so timeout 300 python tools/trace_waits.py 32768 4
done
unset LTL_U8_CELLS
for v in X8 base X8 base; do
  if [[ $v == base ]]; then unset LTL_LIB; else export LTL_LIB=build/ab/$v.so; fi
  echo "== $v"; timeout 300 python tools/pk_time.py 16384 cat; timeout 300 python tools/pk_time.py 32768 cat
done
unset LTL_LIB
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ltl_tc_step -s 3 -c 1 \
  -o gpurun_out/prof_pk_32768 -f python tools/pk_time.py 32768 cat > gpurun_out/ncu_pk.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/prof_pk_32768.ncu-rep --page details --csv 2>/dev/null | grep -E 'Duration|DRAM Throughput|Memory Throughput|Compute \(SM\)|Issue Slots|Registers|Executed Ipc' | head -20
