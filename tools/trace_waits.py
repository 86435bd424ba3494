"""Per-site mbarrier wait cycles of CTA 0 over one traced step launch (trace
build: LTL_NVCC_FLAGS=-DLTL_TC_TRACE_BUILD bash tools/ab_build.sh TR=WORKTREE,
then LTL_LIB=build/ab/TR.so python tools/trace_waits.py n gens [skip]).
Sites (ltl_tc.cu LTL_WAIT): 0 producer x_empty, 1 pass-1 x_full, 2 pass-1
slot_empty, 3-6 convert d1_full, 7 pass-2 a2_full, 8 pass-2 d2_empty, 9-16
output d2_full, 17 producer unit-flag waits (sweep).  Also the launch's
duration from the per-CTA start/end stamps (ns)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
gens = int(sys.argv[2]) if len(sys.argv) > 2 else 10
path = os.path.abspath(f"gpurun_out/trace_{n}_{gens}_{os.environ.get('LTL_NO_PERSIST', 'p')}.csv")
os.makedirs("gpurun_out", exist_ok=True)
os.environ["LTL_TC_TRACE"] = path
os.environ.setdefault("LTL_TC_TRACE_SKIP", sys.argv[3] if len(sys.argv) > 3 else "2")
from paper_2406_17284_b200 import ltl  # noqa: E402

t = ltl.DeviceTorus(rows=n, cols=n)
t.init_random(0.21, 1)
t.run("R5,C2,M1,S34..58,B34..45,NM", 2)      # warm (launches 0.. not traced)
t.run("R5,C2,M1,S34..58,B34..45,NM", gens)
rows = [[int(v) for v in line.split(",")] for line in open(path)]
units = sum(1 for v in rows[1] if v)  # p1 issue stamps (first 256)
starts = [v for v in rows[14] if v]
ends = [v for v in rows[15] if v]
span_us = (max(ends) - min(starts)) / 1e3 if starts and ends else 0
print(f"n={n} gens={gens} persist={'no' if os.environ.get('LTL_NO_PERSIST') else 'auto'} "
      f"launch span {span_us:.1f} us, CTAs {len(starts)}")
names = ["prod x_empty", "p1 x_full", "p1 slot_empty", "cv d1 w2", "cv d1 w3", "cv d1 w4", "cv d1 w5",
         "p2 a2_full", "p2 d2_empty"] + [f"out d2 w{w}" for w in range(6, 14)] + ["prod flags"]
w = rows[13]
for i, nm in enumerate(names):
    print(f"  {i:2d} {nm:14s} {w[i]:14d} cycles")
