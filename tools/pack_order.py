import sys
sys.path.insert(0, '.')
from paper_2406_17284_b200 import ltl
pre = ltl.ltl_presets()
with ltl.DeviceTorus(rows=32768, cols=32768) as t:
    for r in (2, 1, 2, 1, 16, 15, 16):
        name, rule, dens = pre[r - 1]
        t.init_random(dens, 1)
        tot, _ = t.time(rule, 10, 3, engine="pack")
        print(r, name, round(tot / 10 * 1000, 1), "us/gen", flush=True)
    t.init_random(0.5, 1)
    tot, _ = t.time("R1,C2,M0,S2..3,B3..3,NM", 10, 3, engine="pack"); print("life d0.5", round(tot/10*1000,1))
    t.init_random(0.5, 1)
    tot, _ = t.time("R2,C2,M0,S7..12,B8..11,NM", 10, 3, engine="pack"); print("r2 rule d0.5", round(tot/10*1000,1))
