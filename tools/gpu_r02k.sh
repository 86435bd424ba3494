#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "criterion1 or rectangular or large_grid" > gpurun_out/pytest_k.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_k.log
timeout 900 python bench.py --engine pack --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_pack_k.json 2>/dev/null; echo "bench pack rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_c2_pack_k.json').read().splitlines()[-1])
print('pack', ' '.join('r%d:%.3g(%.2f)'%(p['r'],p['cell_updates_per_s'],p['hbm_frac']) for p in d['per_radius']))"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ltl_tc_step -s 1 -c 1 -o gpurun_out/prof_tc_16384_persist -f python bench.py --workload c1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c1.log 2>&1; echo "ncu c1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pack_kernel -s 3 -c 1 -o gpurun_out/prof_pack_r1d -f python bench.py --engine pack --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_pack1d.log 2>&1; echo "ncu pack rc=$?"
