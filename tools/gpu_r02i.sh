#!/bin/bash
set -u
mkdir -p gpurun_out
./build/cpp_e2e 16384 20 > gpurun_out/cpp_e2e_i.txt 2>&1; echo "cpp_e2e rc=$?"; cat gpurun_out/cpp_e2e_i.txt
./paper_2406_17284_b200/bin/catbench bench --rule R5,C2,M1,S34..58,B34..45,NM --density 0.21 --n 16384 --steps 20 --engines cat,base,pack --max-realizations 8 --target-stderr 1 > gpurun_out/cli_bench_i.csv 2>&1; echo "cli bench rc=$?"; cat gpurun_out/cli_bench_i.csv
timeout 2400 python -m pytest tests -q -m gpu -x -rs --deselect tests/test_gpu_large.py > gpurun_out/pytest_i.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_i.log
