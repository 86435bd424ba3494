"""Chained (total) vs isolated (events around every launch) time per
generation of the Cat step (ltl_time's two passes).  python tools/pk_time2.py n [engine]"""
import sys

sys.path.insert(0, ".")
from paper_2406_17284_b200 import ltl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
eng = sys.argv[2] if len(sys.argv) > 2 else "cat"
with ltl.DeviceTorus(n=n) as t:
    t.init_random(0.3, 1)
    for rule in ("R1,C2,M0,S2..3,B3..3,NM", "R5,C2,M1,S34..58,B34..45,NM"):
        tot, ker = t.time(rule, 40, warmup=5, engine=eng)
        print(f"n={n} {rule[:3]} chained {tot / 40 * 1e3:7.1f} us/gen  isolated {ker / 40 * 1e3:7.1f} us/gen", flush=True)
