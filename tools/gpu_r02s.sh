#!/bin/bash
# CUDA-core engines with the byte-lane rule (Moore r <= 3, VN r <= 15):
# parity (all engines), then the configs[2] per-radius tables of pack / base.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_parity_s.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/pytest_parity_s.log
for e in pack base; do
  timeout 900 python bench.py --engine $e --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_${e}_s.json 2>/dev/null; echo "bench $e rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/bench_c2_${e}_s.json').read().splitlines()[-1])
print('$e', ' '.join('r%d:%.3g(%.2f)'%(p['r'],p['cell_updates_per_s'],p['hbm_frac']) for p in d['per_radius']))"
done
