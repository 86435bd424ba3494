#!/bin/bash
# Round-2 first GPU session: host facts, i8 peak, GPU tests, the configs[2]
# bench line + reference arm, launch list and one ncu --set full capture.
set -u
mkdir -p gpurun_out
(nvidia-smi; free -g; nproc; lscpu | head -20) > gpurun_out/host.txt 2>&1
timeout 120 ./build/ubench_mma --peak gpurun_out/ubench_mma_peak.json > gpurun_out/ubench_mma_peak.txt 2>&1
echo "ubench rc=$?"; cat gpurun_out/ubench_mma_peak.txt
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?"
tail -c 4000 gpurun_out/bench_c2.json; tail -5 gpurun_out/bench_c2.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_c2.json 2> gpurun_out/ref_c2.err; echo "ref rc=$?"
tail -c 2000 gpurun_out/ref_c2.json; tail -5 gpurun_out/ref_c2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ltl_tc_step -s 5 -c 1 \
  -o gpurun_out/prof_tc_32768 -f python bench.py --steps 5 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
