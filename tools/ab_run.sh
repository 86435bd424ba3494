#!/bin/bash
# Interleaved A/B timing of libraries built by tools/ab_build.sh (run on the GPU box):
#   bash tools/ab_run.sh "--n 16384 --steps 200" 3 A B
set -u
args=$1; reps=$2; shift 2
for i in $(seq "$reps"); do
  for v in "$@"; do
    echo -n "$v: "
    LTL_LIB=build/ab/$v.so timeout 300 python bench.py $args --no-cpu-baseline 2>/dev/null | python tools/bench_line.py
  done
done
