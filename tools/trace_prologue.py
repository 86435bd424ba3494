"""Per-CTA prologue / PDL-wait / body times of one traced step launch inside a
chain of per-generation launches (trace build: LTL_NVCC_FLAGS=-DLTL_TC_TRACE_BUILD
bash tools/ab_build.sh TR=WORKTREE; LTL_LIB=build/ab/TR.so python tools/trace_prologue.py n)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
path = os.path.abspath(f"gpurun_out/trace_prologue_{n}.csv")
os.makedirs("gpurun_out", exist_ok=True)
os.environ["LTL_TC_TRACE"] = path
os.environ["LTL_TC_TRACE_SKIP"] = "4"
os.environ["LTL_NO_PERSIST"] = "1"
from paper_2406_17284_b200 import ltl  # noqa: E402

t = ltl.DeviceTorus(rows=n, cols=n)
t.init_random(0.21, 1)
t.run("R5,C2,M1,S34..58,B34..45,NM", 8)
rows = [[int(v) for v in line.split(",")] for line in open(path)]
ent, pro, go, end = rows[10], rows[12], rows[14], rows[15]
ctas = [i for i in range(256) if ent[i]]
t0 = min(ent[i] for i in ctas)
pl = sorted((pro[i] - ent[i]) / 1e3 for i in ctas)
print(f"n={n} CTAs {len(ctas)}: entry spread {(max(ent[i] for i in ctas) - t0) / 1e3:.1f} us, "
      f"prologue median {pl[len(pl) // 2]:.2f} max {pl[-1]:.2f} us, "
      f"first body start {(min(go[i] for i in ctas) - t0) / 1e3:.1f} us, last {(max(go[i] for i in ctas) - t0) / 1e3:.1f} us, "
      f"first end {(min(end[i] for i in ctas) - t0) / 1e3:.1f} us, last end {(max(end[i] for i in ctas) - t0) / 1e3:.1f} us")
