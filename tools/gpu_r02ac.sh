#!/bin/bash
# After the bit-packed transfers: the whole GPU suite + smoke, the bench line
# (e2e), the C++ drop-in end to end.
set -u
mkdir -p gpurun_out
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python tools/bench_line.py < gpurun_out/bench.json
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().splitlines()[-1]); print('e2e', d['e2e'])"
g++ -std=c++20 -O2 -Iinclude tools/cpp_e2e.cpp -Lpaper_2406_17284_b200 -lltl_b200 -Wl,-rpath,$PWD/paper_2406_17284_b200 -o build/cpp_e2e && ./build/cpp_e2e 16384 20 > gpurun_out/cpp_e2e.txt 2>&1; echo "cpp_e2e rc=$?"; cat gpurun_out/cpp_e2e.txt | tail -8
