#!/bin/bash
# Wide radius (32-row boxes) with the dynamic remainder (W1) vs static (W0).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py -q -x > gpurun_out/pytest_w.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/pytest_w.log
for v in W0 W1 W0 W1; do
  echo "== $v"; LTL_LIB=build/ab/$v.so timeout 600 python bench.py --workload wide --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python tools/bench_line.py
done
