#!/bin/bash
# ncu of the pack engine at r = 1 and r = 2 (configs[2] sweep launches 4 and 15).
set -u
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pack_kernel -s 3 -c 1 -o gpurun_out/prof_pack_r1t -f python bench.py --engine pack --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_pack1t.log 2>&1; echo "ncu pack r1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pack_kernel -s 9 -c 1 -o gpurun_out/prof_pack_r2t -f python bench.py --engine pack --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_pack2t.log 2>&1; echo "ncu pack r2 rc=$?"
