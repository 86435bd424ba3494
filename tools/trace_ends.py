"""CTA end-time spread of one per-launch step (trace build TR2), excluding the
instrumented CTA 0.  LTL_LIB=build/ab/TR2.so python tools/trace_ends.py n"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
path = os.path.abspath(f"gpurun_out/trace_ends_{n}.csv")
os.makedirs("gpurun_out", exist_ok=True)
os.environ.update(LTL_TC_TRACE=path, LTL_TC_TRACE_SKIP="4", LTL_NO_PERSIST="1")
from paper_2406_17284_b200 import ltl  # noqa: E402

t = ltl.DeviceTorus(rows=n, cols=n)
t.init_random(0.21, 1)
t.run("R5,C2,M1,S34..58,B34..45,NM", 8)
rows = [[int(v) for v in line.split(",")] for line in open(path)]
go, end = rows[14], rows[15]
ctas = [i for i in range(1, 256) if go[i]]
t0 = min(go[i] for i in ctas)
e = [(end[i] - t0) / 1e3 for i in ctas]
print(f"n={n}: body end mean {statistics.mean(e):.1f} median {statistics.median(e):.1f} "
      f"max {max(e):.1f} us; slowest {sorted(ctas, key=lambda i: -end[i])[:10]}")
