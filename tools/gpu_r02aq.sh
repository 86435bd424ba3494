#!/bin/bash
# compute-sanitizer over every engine / path on the current tree (cp.async stencils, 4-bit cells, bit transfers).
set -u
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize.py > gpurun_out/sanitizer_$tool.txt 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/sanitizer_$tool.txt
done
