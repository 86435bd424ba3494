#!/bin/bash
set -u
cat > /tmp/c1.py <<'PY'
import sys
sys.path.insert(0, '.')
from paper_2406_17284_b200 import ltl
with ltl.DeviceTorus(rows=16384, cols=16384) as t:
    t.init_random(0.21, 1)
    tot, ker = t.time("R5,C2,M1,S34..58,B34..45,NM", 200, 10)
    print(round(tot / 200 * 1000, 2), "us/gen", t.time_launches(), "launches", flush=True)
PY
for v in "" "LTL_SWEEP_UNITS=8" "LTL_SWEEP_UNITS=16" "LTL_SWEEP_UNITS=32" "LTL_SWEEP_UNITS=64" "LTL_SWEEP_UNITS=128" "LTL_TC_GRID=128" "LTL_TC_GRID=128 LTL_SWEEP_UNITS=16" "LTL_TC_GRID=144" "LTL_NO_PERSIST=1" ""; do
  echo -n "[$v] "; env $v python /tmp/c1.py
done
