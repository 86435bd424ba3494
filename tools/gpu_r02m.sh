#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_ref_suites.py tests/test_cli.py -q -m gpu -rs > gpurun_out/pytest_m.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_m.log
./build/ref_suites/acceptance > gpurun_out/acceptance_m.txt 2>&1; echo "acceptance rc=$?"; cat gpurun_out/acceptance_m.txt
./build/ref_suites/acceptance --soft > gpurun_out/acceptance_soft_m.txt 2>&1; echo "acceptance --soft rc=$?"; tail -3 gpurun_out/acceptance_soft_m.txt
