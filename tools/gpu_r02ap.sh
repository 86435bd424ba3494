#!/bin/bash
# CUDA-core engines, cp.async loads, no CTA caps: parity + bench lines of both engines, ncu of pack r=1.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -q -x -k "criterion1 or anchors or rectangular or stencil or engines_agree or halo" > gpurun_out/pytest_st2.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pytest_st2.log
for e in pack base; do
  timeout 900 python bench.py --engine $e --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_$e.json 2>/dev/null; echo "bench $e rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/bench_c2_$e.json').read().splitlines()[-1])
print('$e', ' '.join('r%d:%.3g(%.2f)'%(p['r'],p['cell_updates_per_s'],p['hbm_frac']) for p in d['per_radius']))"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pack_kernel -s 3 -c 1 -o gpurun_out/prof_pack_r1_f -f python bench.py --engine pack --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_pack1f.log 2>&1; echo "ncu pack r1 rc=$?"
