#!/bin/bash
# CUDA-core engines with cp.async tile loads: CTAs per SM re-tuned (pack SMEM floor, base padding).
set -u
mkdir -p gpurun_out
run() {  # engine label env...
  local e=$1 lab=$2; shift 2
  env "$@" timeout 600 python bench.py --engine $e --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_t.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/b_t.json').read().splitlines()[-1])
print('$e $lab', ' '.join('r%d:%.3g(%.2f)'%(p['r'],p['cell_updates_per_s'],p['hbm_frac']) for p in d['per_radius'] if p['r'] in (1,2,3,4,8,12,16)))"
}
for i in 1 2; do
  run pack floor0 LTL_PACK_MIN_SMEM=0
  run pack floor47k LTL_PACK_MIN_SMEM=47000
  run pack floor60k LTL_PACK_MIN_SMEM=60000
  run base pad0 LTL_BASE_PAD_SMEM=0
  run base pad4k LTL_BASE_PAD_SMEM=4000
  run base pad10k LTL_BASE_PAD_SMEM=10000
done
