#!/bin/bash
# CUDA-core engines after the byte-lane rule + CTA caps: parity, per-radius
# tables; the wide-radius bench line and its ncu on the current binary.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py -q -x > gpurun_out/pytest_v.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/pytest_v.log
for e in pack base; do
  timeout 900 python bench.py --engine $e --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_${e}_v.json 2>/dev/null; echo "bench $e rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/bench_c2_${e}_v.json').read().splitlines()[-1])
print('$e', ' '.join('r%d:%.3g(%.2f)'%(p['r'],p['cell_updates_per_s'],p['hbm_frac']) for p in d['per_radius']))"
done
timeout 900 python bench.py --workload wide --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_wide_v.json 2> gpurun_out/bench_wide_v.err; echo "bench wide rc=$?"
python tools/bench_line.py < gpurun_out/bench_wide_v.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ltl_tc_step -s 5 -c 1 \
  -o gpurun_out/prof_tc_wide_32768_v -f python bench.py --workload wide --steps 5 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_wide_v.log 2>&1; echo "ncu wide rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pack_kernel -s 3 -c 1 -o gpurun_out/prof_pack_r1v -f python bench.py --engine pack --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_pack1v.log 2>&1; echo "ncu pack r1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:base_kernel -s 3 -c 1 -o gpurun_out/prof_base_r1v -f python bench.py --engine base --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_base1v.log 2>&1; echo "ncu base r1 rc=$?"
