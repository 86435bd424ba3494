"""Prologue stage times per CTA (build: LTL_NVCC_FLAGS="-DLTL_TC_TRACE_BUILD
-DLTL_PROLOGUE_TRACE" bash tools/ab_build.sh TP=WORKTREE; LTL_LIB=build/ab/TP.so
python tools/trace_prologue2.py n)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
path = os.path.abspath(f"gpurun_out/trace_prologue2_{n}.csv")
os.makedirs("gpurun_out", exist_ok=True)
os.environ["LTL_TC_TRACE"] = path
os.environ["LTL_TC_TRACE_SKIP"] = "4"
os.environ["LTL_NO_PERSIST"] = "1"
from paper_2406_17284_b200 import ltl  # noqa: E402

t = ltl.DeviceTorus(rows=n, cols=n)
t.init_random(0.21, 1)
t.run("R5,C2,M1,S34..58,B34..45,NM", 8)
rows = [[int(v) for v in line.split(",")] for line in open(path)]
ctas = [i for i in range(256) if rows[10][i]]
stages = [("band tiles", 10, 0), ("barriers + TMEM alloc", 0, 1), ("A table -> TMEM", 1, 2),
          ("to prologue end", 2, 12), ("PDL wait", 12, 14)]
for name, a, b in stages:
    d = [(rows[b][i] - rows[a][i]) / 1e3 for i in ctas]
    print(f"{name:24s} median {statistics.median(d):6.2f} us  max {max(d):6.2f} us")
