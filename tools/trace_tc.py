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

names = ["tma issue", "p1 issue", "-", "-", "p2 issue", "-", "-", "-", "-", "-", "-", "out stored"]
rows = [[int(v) for v in line.split(",")] for line in open(path)]
t0 = min(v for r in rows for v in r if v > 0)
print("chunk " + " ".join(f"{nm[:12]:>12s}" for nm in names))
for k in range(40):
    print(f"{k:5d} " + " ".join(f"{(rows[e][k] - t0) if rows[e][k] else -1:12d}" for e in range(12)))
