#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "criterion1 or rectangular or large_grid or refreshes or all_alive" > gpurun_out/pytest_o.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_o.log
timeout 900 python bench.py --engine pack --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_pack_o.json 2>/dev/null; echo "bench pack rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_c2_pack_o.json').read().splitlines()[-1])
print('pack', ' '.join('r%d:%.3g(%.2f)'%(p['r'],p['cell_updates_per_s'],p['hbm_frac']) for p in d['per_radius']))"
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize.py > gpurun_out/san_memcheck_o.txt 2>&1; echo "memcheck rc=$?"; tail -2 gpurun_out/san_memcheck_o.txt
