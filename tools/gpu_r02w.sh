set -u
# 4-bit-cell probe (tools/ubench_fp4b.cu), smoke and the whole GPU suite.
mkdir -p gpurun_out
timeout 60 ./build/ubench_fp4b > gpurun_out/fp4b.txt 2>&1; echo "probe rc=$?"; cat gpurun_out/fp4b.txt
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
