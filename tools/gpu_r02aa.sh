#!/bin/bash
# 4-bit cells as the opt-in engine: its GPU tests, the u8 suite's parity core,
# the bench line of each engine on configs[2].
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_4bit.py -q -x > gpurun_out/pytest_4bit.log 2>&1; echo "4bit tests rc=$?"; tail -3 gpurun_out/pytest_4bit.log
for e in cat cat-4bit; do
  timeout 900 python bench.py --engine $e --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2_$e.json 2> gpurun_out/bench_c2_$e.err; echo "bench $e rc=$?"
  python tools/bench_line.py < gpurun_out/bench_c2_$e.json
done
