"""A/B timing helper (GPU box): per-generation time of three rules at 16384^2
(persistent sweep) and 32768^2 (a launch per generation) for the library
LTL_LIB points at.   LTL_LIB=build/ab/A.so python tools/ab_sizes.py A"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_17284_b200 import ltl  # noqa: E402

out = []
for n, steps in ((16384, 200), (32768, 40)):
    with ltl.DeviceTorus(n=n) as t:
        for text, dens in (("R5,C2,M1,S34..58,B34..45,NM", 0.21), ("R1,C2,M0,S2..3,B3..3,NM", 0.07),
                           ("R16,C2,M0,S170..296,B170..300,NM", 0.26)):
            t.init_random(dens, 1)
            tot, ker = t.time(text, steps, 10)
            out.append("%d r%s %.2f us" % (n, text[1:text.index(',')], tot / steps * 1e3))
print(sys.argv[1] if len(sys.argv) > 1 else "", " | ".join(out), flush=True)
