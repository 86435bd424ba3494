# full GPU check: parity suite, default bench line, 32768 line (GPU box)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 300 python bench.py --n 32768 --steps 300 --no-cpu-baseline > gpurun_out/bench_32768.json 2>> gpurun_out/bench_default.err
