#!/bin/bash
set -u
mkdir -p gpurun_out
export LTL_LIB=build/ab/TR.so
python tools/trace_waits.py 16384 10 1
LTL_NO_PERSIST=1 python tools/trace_waits.py 16384 10 4
python tools/trace_waits.py 32768 4 4
