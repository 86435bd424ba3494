mkdir -p gpurun_out
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 300 python bench.py --steps 300 --no-cpu-baseline > gpurun_out/b16.json 2>gpurun_out/b.err
timeout 300 python bench.py --n 32768 --steps 100 --no-cpu-baseline > gpurun_out/b32.json 2>>gpurun_out/b.err
