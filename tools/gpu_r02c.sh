#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -rs -k "fault or determinism or cli or ref_suite or persistent or ring" > gpurun_out/pytest_gpu_c.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu_c.log
timeout 1800 python -m pytest tests/test_gpu_large.py -q -rs > gpurun_out/pytest_large_c.log 2>&1; echo "large rc=$?"
tail -15 gpurun_out/pytest_large_c.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize.py > gpurun_out/san_memcheck.txt 2>&1; echo "memcheck rc=$?"; tail -5 gpurun_out/san_memcheck.txt
