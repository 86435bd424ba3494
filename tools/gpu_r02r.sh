#!/bin/bash
# A/B (interleaved) of two library builds in build/ab/: tools/ab_sizes.py.
set -u
mkdir -p gpurun_out
for i in 1 2 3; do for v in ${AB:-A B}; do LTL_LIB=build/ab/$v.so timeout 300 python tools/ab_sizes.py $v; done; done 2>&1 | tee gpurun_out/ab_r.txt
