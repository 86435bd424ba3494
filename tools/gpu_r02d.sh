#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_ref_suites.py -q -m gpu -rs > gpurun_out/pytest_acc_d.log 2>&1; echo "acc rc=$?"; tail -5 gpurun_out/pytest_acc_d.log
./build/ref_suites/acceptance > gpurun_out/acceptance_d.txt 2>&1; echo "acceptance rc=$?"; cat gpurun_out/acceptance_d.txt
for v in "" "LTL_FORCE_PERSIST=1" "LTL_FORCE_PERSIST=1 LTL_SWEEP_UNITS=1" "LTL_FORCE_PERSIST=1 LTL_SWEEP_UNITS=2"; do
  env $v timeout 300 python bench.py --workload c0 --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/c0.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/c0.json').read().splitlines()[-1]); print('c0 [$v]', round(d['ms_per_step']*1000,2),'us/gen', d['gpu_launches'],'launches')"
done
timeout 300 python bench.py --workload c1 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/c1_d.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/c1_d.json').read().splitlines()[-1]); print('c1', round(d['ms_per_step']*1000,2),'us/gen', d['value'], d['gpu_launches'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pack_kernel -s 3 -c 1 -o gpurun_out/prof_pack_r1 -f python bench.py --engine pack --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_pack1.log 2>&1; echo "ncu pack r1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pack_kernel -s 3 -c 1 -o gpurun_out/prof_pack_r16 -f python bench.py --engine pack --workload c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_pack16.log 2>&1; echo "ncu pack r16 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:base_kernel -s 3 -c 1 -o gpurun_out/prof_base_r1 -f python bench.py --engine base --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_base1.log 2>&1; echo "ncu base r1 rc=$?"
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize.py > gpurun_out/san_racecheck.txt 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/san_racecheck.txt
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize.py > gpurun_out/san_synccheck.txt 2>&1; echo "synccheck rc=$?"; tail -3 gpurun_out/san_synccheck.txt
