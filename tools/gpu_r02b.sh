#!/bin/bash
# Round-2 session b: full GPU test suite (new engines, fault parity, reference
# suites, CLI), stencil radius sweeps, C++ end-to-end timing.
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rs > gpurun_out/pytest_gpu_b.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu_b.log
for e in base pack; do
  timeout 900 python bench.py --engine $e --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_$e.json 2> gpurun_out/bench_c2_$e.err; echo "bench $e rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/bench_c2_$e.json').read().splitlines()[-1])
print('$e', ' '.join('r%d:%.3g(%.2f)'%(p['r'],p['cell_updates_per_s'],p['hbm_frac']) for p in d['per_radius']))"
done
N=16384
for i in 1 2; do
  timeout 600 ./paper_2406_17284_b200/bin/catbench run --rule R5,C2,M1,S34..58,B34..45,NM --density 0.21 --n $N --steps 20 > gpurun_out/cli_e2e_$i.txt 2>&1; echo "cli rc=$?"; cat gpurun_out/cli_e2e_$i.txt
done
