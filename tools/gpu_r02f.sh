#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x -rs --deselect tests/test_gpu_large.py > gpurun_out/pytest_f.log 2>&1; echo "pytest rc=$?"; tail -6 gpurun_out/pytest_f.log
for e in base pack; do
  timeout 900 python bench.py --engine $e --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_$e.json 2> gpurun_out/bench_c2_$e.err; echo "bench $e rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/bench_c2_$e.json').read().splitlines()[-1])
print('$e', ' '.join('r%d:%.3g(%.2f)'%(p['r'],p['cell_updates_per_s'],p['hbm_frac']) for p in d['per_radius']))"
done
cat > /tmp/small.py <<'PY'
import sys, json
sys.path.insert(0, '.')
from paper_2406_17284_b200 import ltl
for n in (1024, 2048, 4096):
    with ltl.DeviceTorus(rows=n, cols=n) as t:
        t.init_random(0.5, 1)
        tot, ker = t.time("R1,C2,M0,S2..3,B3..3,NM", 200, 20)
        print(n, round(tot / 200 * 1000, 2), "us/gen", t.time_launches(), "launches", flush=True)
PY
echo "small default"; python /tmp/small.py
echo "small LTL_NO_SMALL_PERSIST"; LTL_NO_SMALL_PERSIST=1 python /tmp/small.py
echo "small LTL_FORCE_PERSIST"; LTL_FORCE_PERSIST=1 python /tmp/small.py
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pack_kernel -s 3 -c 1 -o gpurun_out/prof_pack_r1c -f python bench.py --engine pack --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_pack1c.log 2>&1; echo "ncu pack r1 rc=$?"
