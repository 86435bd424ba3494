#!/bin/bash
set -u
mkdir -p gpurun_out
./paper_2406_17284_b200/bin/catbench bench --rule R5,C2,M1,S34..58,B34..45,NM --density 0.21 --n 16384 --steps 20 --engines cat --max-realizations 5 --target-stderr 1 > gpurun_out/cli_bench_g.csv 2>&1; echo "cli bench rc=$?"; cat gpurun_out/cli_bench_g.csv
timeout 600 python bench.py --workload c1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c1_g.json 2>&1; echo "c1 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/c1_g.json').read().splitlines()[-1]); print('c1 value', d['value'], 'e2e', d['e2e'])"
timeout 900 python bench.py --dist --workload c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c4_dist_g.json 2> gpurun_out/c4_dist_g.err; echo "c4 dist rc=$?"; tail -c 1500 gpurun_out/c4_dist_g.json; tail -3 gpurun_out/c4_dist_g.err
