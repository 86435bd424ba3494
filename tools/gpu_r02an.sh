#!/bin/bash
# CUDA-core engines with cp.async tile loads (STNEW) vs register-staged (STOLD): parity, per-radius.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "criterion1 or anchors or rectangular" > gpurun_out/pytest_st.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pytest_st.log
for v in STOLD STNEW STOLD STNEW; do
  for e in pack base; do
    LTL_LIB=build/ab/$v.so timeout 600 python bench.py --engine $e --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_${v}_$e.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/b_${v}_$e.json').read().splitlines()[-1])
print('$v $e', ' '.join('r%d:%.3g(%.2f)'%(p['r'],p['cell_updates_per_s'],p['hbm_frac']) for p in d['per_radius'] if p['r'] in (1,2,3,4,8,12,16)))"
  done
done
