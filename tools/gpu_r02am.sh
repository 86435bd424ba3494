#!/bin/bash
# Final validation of the current tree: smoke, the whole GPU suite, the bench line.
set -u
mkdir -p gpurun_out
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python tools/bench_line.py < gpurun_out/bench.json
python -c "import json; d=json.loads(open('gpurun_out/bench.json').read().splitlines()[-1]); print('e2e %.3e'%d['e2e']['value'], d['e2e']['h2d_bytes_per_step'], 'launches', d['gpu_launches'])"
