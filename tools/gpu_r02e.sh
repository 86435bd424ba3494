#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_cli.py -q -m gpu -x -k "criterion1 or anchors or rectangular or large_grid or refreshes or all_alive or verify" > gpurun_out/pytest_e.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_e.log
for e in base pack; do
  timeout 900 python bench.py --engine $e --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_$e.json 2> gpurun_out/bench_c2_$e.err; echo "bench $e rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/bench_c2_$e.json').read().splitlines()[-1])
print('$e', ' '.join('r%d:%.3g(%.2f)'%(p['r'],p['cell_updates_per_s'],p['hbm_frac']) for p in d['per_radius']))"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pack_kernel -s 3 -c 1 -o gpurun_out/prof_pack_r1b -f python bench.py --engine pack --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_pack1b.log 2>&1; echo "ncu pack r1 rc=$?"
