#!/bin/bash
# Dynamic remainder only after whole-band rounds (DYN2) vs static (STAT): timing, then the whole GPU suite and the bench line.
set -u
mkdir -p gpurun_out
for v in STAT DYN2 STAT DYN2; do
  echo "== $v"
  LTL_LIB=build/ab/$v.so timeout 300 python tools/pk_time.py 32768 cat cat-4bit
  LTL_LIB=build/ab/$v.so timeout 300 python tools/pk_time.py 8192 cat
done
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python tools/bench_line.py < gpurun_out/bench.json
timeout 900 python bench.py --workload wide --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_wide.json 2> gpurun_out/bench_wide.err; echo "bench wide rc=$?"
python tools/bench_line.py < gpurun_out/bench_wide.json
