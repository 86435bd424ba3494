#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_j.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_j.log
timeout 1800 python -m pytest tests/test_gpu_large.py -q -rs > gpurun_out/pytest_large_j.log 2>&1; echo "large rc=$?"; tail -5 gpurun_out/pytest_large_j.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_j.json 2> gpurun_out/bench_j.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open('gpurun_out/bench_j.json').read().splitlines()[-1])
print({k: d[k] for k in ('value', 'ms_per_step', 'gpu_launches', 'aggregate_value')})
print('roofline', {k: d['roofline'][k] for k in ('achieved', 'frac', 'traffic', 'kernel_ms_per_generation', 'mma_frac')})
print('e2e', d['e2e']['value'], 'cpu', d.get('cpu_baseline', {}).get('value'), d['clocks'])
PY
