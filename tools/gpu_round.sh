#!/bin/bash
# One GPU session: build, smoke, GPU tests, bench, ncu launch list + one full capture.
# Usage (from the repo root, under gpurun): bash tools/gpu_round.sh [tests|bench|ncu|all]
set -u
mkdir -p gpurun_out
what=${1:-all}
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
if [[ $what == all || $what == tests ]]; then
  timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
  timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -5 gpurun_out/pytest_gpu.log
fi
if [[ $what == all || $what == bench ]]; then
  timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
  tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
fi
if [[ $what == all || $what == ncu ]]; then
  # launch list of the default bench command (shorter run); the timed loop
  # is launch 2 of ltl_tc_step (after the warm-up launch)
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_bench.log 2>&1; echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ltl_tc_step -s 1 -c 1 \
    -o gpurun_out/prof_tc -f python bench.py --steps 20 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
  # one generation per launch (32768^2 policy) for comparison
  LTL_NO_PERSIST=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:ltl_tc_step -s 5 -c 1 \
    -o gpurun_out/prof_tc_perlaunch -f python bench.py --steps 10 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_full_pl.log 2>&1; echo "ncu full (per launch) rc=$?"
fi
