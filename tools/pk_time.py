"""Device time per generation of the Cat step, 4-bit vs u8 cells (A/B on one
box; LTL_LIB selects a library build).  python tools/pk_time.py [n] [engine...]"""
import sys

sys.path.insert(0, ".")
from paper_2406_17284_b200 import ltl  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
engines = sys.argv[2:] or ["cat", "cat-4bit"]
for rule in ("R1,C2,M0,S2..3,B3..3,NM", "R5,C2,M1,S34..58,B34..45,NM"):
    for eng in engines:
        with ltl.DeviceTorus(n=n) as t:
            t.init_random(0.3, 1)
            tot, _ = t.time(rule, 20, warmup=5, engine=eng)
            print(f"n={n} {rule[:3]} {eng:8s} {tot / 20 * 1e3:8.1f} us/gen "
                  f"{n * n * 20 / (tot * 1e-3):.3e} cell updates/s", flush=True)
