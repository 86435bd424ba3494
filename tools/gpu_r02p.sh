#!/bin/bash
# Wide-radius bench line + ncu of the current binary's step kernels (the
# template now carries the box halo: ltl_tc_step_kernel<16,..> / <32,..>).
set -u
mkdir -p gpurun_out
timeout 900 python bench.py --workload wide --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_wide_p.json 2> gpurun_out/bench_wide_p.err; echo "bench wide rc=$?"
python tools/bench_line.py < gpurun_out/bench_wide_p.json; tail -2 gpurun_out/bench_wide_p.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ltl_tc_step -s 5 -c 1 \
  -o gpurun_out/prof_tc_wide_32768 -f python bench.py --workload wide --steps 5 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_wide.log 2>&1; echo "ncu wide rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ltl_tc_step -s 5 -c 1 \
  -o gpurun_out/prof_tc_32768_p -f python bench.py --steps 5 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_c2_p.log 2>&1; echo "ncu c2 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches_c2_p.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_launch_p.log 2>&1; echo "ncu launches rc=$?"
