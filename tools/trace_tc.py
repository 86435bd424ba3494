"""Capture and print the tcgen05 pipeline timeline of CTA 0 (debug aid).
Usage on the GPU box: python tools/trace_tc.py [n] [rule]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
path = os.path.abspath("gpurun_out/tc_trace.csv")
os.makedirs("gpurun_out", exist_ok=True)
os.environ["LTL_TC_TRACE"] = path
from paper_2406_17284_b200 import ltl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
rule = sys.argv[2] if len(sys.argv) > 2 else "R5,C2,M1,S34..58,B34..45,NM"
t = ltl.DeviceTorus(rows=n, cols=n)
t.init_random(0.21, 1)
t.time(rule, 2, 0)

names = ["tma issue", "p1 issue", "cv start", "cv read", "p2 issue", "out0 go", "out0 read", "out1 go", "-", "-", "-", "out stored"]
rows = [[int(v) for v in line.split(",")] for line in open(path)]
t0 = min(v for r in rows for v in r if v > 0)
print("chunk " + " ".join(f"{nm[:12]:>12s}" for nm in names))
for k in range(40):
    print(f"{k:5d} " + " ".join(f"{(rows[e][k] - t0) if rows[e][k] else -1:12d}" for e in range(12)))
# steady-state per-unit deltas (units 20..60): stage latencies relative to p1 issue
import statistics
def d(e1, e2, k1, k2):
    return rows[e2][k2] - rows[e1][k1]
ks = [k for k in range(20, 60) if all(rows[e][k] for e in (1, 2, 3, 5, 6, 11))]
if ks:
    print("unit period (p1 issue):", statistics.median(rows[1][k + 1] - rows[1][k] for k in ks))
    print("p1 issue -> cv start  :", statistics.median(d(1, 2, k, k) for k in ks))
    print("cv start -> cv read   :", statistics.median(d(2, 3, k, k) for k in ks))
    print("cv read  -> cv done   :", statistics.median(d(3, 8, k, k) for k in ks))
    print("cv done  -> p2 issue s0:", statistics.median(rows[4][2 * k] - rows[8][k] for k in ks))
    print("p2 s1 issue -> p1 issue(k+2):", statistics.median(rows[1][k + 2] - rows[4][2 * k + 1] for k in ks))
    print("cv read  -> p2 issue s0:", statistics.median(rows[4][2 * k] - rows[3][k] for k in ks))
    print("p2 s0 -> out0 go      :", statistics.median(rows[5][k] - rows[4][2 * k] for k in ks))
    print("out0 go -> out0 read  :", statistics.median(d(5, 6, k, k) for k in ks))
    print("out0 go -> stored     :", statistics.median(d(5, 11, k, k) for k in ks))
    print("p1 issue(k) -> p1 issue(k+2):", statistics.median(rows[1][k + 2] - rows[1][k] for k in ks))
print("wait sums (row 13):", rows[13][:20])
