#!/bin/bash
# Final state: sanitizers (incl. the dynamic schedule), the whole GPU suite, smoke, bench, launch list, ncu of the step.
set -u
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize.py > gpurun_out/sanitizer_$tool.txt 2>&1; echo "$tool rc=$?"; tail -1 gpurun_out/sanitizer_$tool.txt
done
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python tools/bench_line.py < gpurun_out/bench.json
python -c "import json; d=json.loads(open('gpurun_out/bench.json').read().splitlines()[-1]); print('e2e %.3e'%d['e2e']['value'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ltl_tc_step -s 5 -c 1 -o gpurun_out/prof_tc_final2 -f python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
