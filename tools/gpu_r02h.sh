#!/bin/bash
set -u
mkdir -p gpurun_out
./build/cpp_e2e 16384 20 > gpurun_out/cpp_e2e_h.txt 2>&1; echo "cpp_e2e rc=$?"; cat gpurun_out/cpp_e2e_h.txt
cat > /tmp/sweep.py <<'PY'
import sys
sys.path.insert(0, '.')
from paper_2406_17284_b200 import ltl
with ltl.DeviceTorus(rows=32768, cols=32768) as t:
    t.init_random(0.21, 1)
    tot, ker = t.time("R5,C2,M1,S34..58,B34..45,NM", 100, 10)
    print(round(tot / 100 * 1000, 1), "us/gen", t.time_launches(), "launches", flush=True)
PY
echo "32768 default"; python /tmp/sweep.py
for u in 12 32 64 128 256; do echo "32768 persist units=$u"; LTL_FORCE_PERSIST=1 LTL_SWEEP_UNITS=$u python /tmp/sweep.py; done
echo "32768 default again"; python /tmp/sweep.py
