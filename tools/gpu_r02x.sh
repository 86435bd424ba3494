#!/bin/bash
# 4-bit cells: packed Cat step vs the u8 Cat step, fault parity, first timings.
set -u
mkdir -p gpurun_out
timeout 1200 python tools/pk_check.py > gpurun_out/pk_check.txt 2>&1; echo "pk_check rc=$?"; tail -40 gpurun_out/pk_check.txt
