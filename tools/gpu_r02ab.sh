#!/bin/bash
# Bit-packed host <-> device transfers: round-trip tests, the suites that move
# grids (snapshots, C++ API, reference suites), e2e A/B (bytes vs bits).
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_transfers.py tests/test_gpu_snapshot.py tests/test_cpp_api.py tests/test_ref_suites.py tests/test_cli.py -q -x -m gpu > gpurun_out/pytest_xfer.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pytest_xfer.log
for v in bits bytes bits bytes; do
  if [[ $v == bytes ]]; then export LTL_BYTE_TRANSFERS=1; else unset LTL_BYTE_TRANSFERS; fi
  timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_e2e_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/bench_e2e_$v.json').read().splitlines()[-1])
print('$v', 'value %.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'], 'agg %.3e'%d['e2e']['aggregate_value'])"
done
