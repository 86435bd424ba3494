#!/bin/bash
# Schedule sweep: kernel time vs units layout (debug knobs of launch_tc_step).
for n in 16384 32768; do
  for cfg in "" "LTL_TC_SEGS=1" "LTL_TC_SEGS=2" "LTL_TC_SEGS=4" "LTL_TC_SEGS=37" "LTL_TC_SEGS=74"; do
    v=$(env $cfg python bench.py --no-cpu-baseline --steps 100 --n $n | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,1), round(d['roofline']['kernel_ms_per_launch']*1000,1))")
    echo "n=$n [$cfg] step_us kernel_us: $v"
  done
done
