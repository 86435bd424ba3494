#!/bin/bash
# Round-2 re-entry check: smoke, the whole -m gpu suite, the bench line.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/host_n.txt 2>&1
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_n.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_n.log
timeout 2400 python -m pytest tests -q -m gpu -x -rs > gpurun_out/pytest_gpu_n.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/pytest_gpu_n.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n.json 2> gpurun_out/bench_n.err; echo "bench rc=$?"
python tools/bench_line.py < gpurun_out/bench_n.json; tail -3 gpurun_out/bench_n.err
