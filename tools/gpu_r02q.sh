#!/bin/bash
# Wide-radius kernel A/B: its tests and the r = 16 / 17..32 timings at 32768^2.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py -q -x -rs > gpurun_out/pytest_wide_q.log 2>&1; echo "wide rc=$?"; tail -3 gpurun_out/pytest_wide_q.log
timeout 300 python - <<'PY' > gpurun_out/wide_timing_q.txt 2>&1
from paper_2406_17284_b200 import ltl
n = 32768
def maj(r, vn=False):
    cells = 4 * r if vn else (2 * r + 1) ** 2 - 1
    return [r, 2, 0, cells // 2, cells, cells // 2 + 1, cells, 1 if vn else 0]
with ltl.DeviceTorus(n=n) as t:
    t.init_random(0.5, 1)
    for rule in (maj(16), maj(17), maj(24), maj(32), maj(32, True)):
        tot, ker = t.time(rule, 20, 5)
        print(rule[0], rule[7], "ms/gen %.4f kernel %.4f cells/s %.3e" % (tot / 20, ker / 20, n * n / (tot / 20) * 1e3))
with ltl.DeviceTorus(n=16384) as t:
    t.init_random(0.5, 1)
    for rule in (maj(16), maj(32)):
        tot, ker = t.time(rule, 50, 5)
        print(16384, rule[0], "ms/gen %.4f cells/s %.3e" % (tot / 50, 16384 ** 2 / (tot / 50) * 1e3))
PY
echo "timing rc=$?"; cat gpurun_out/wide_timing_q.txt
