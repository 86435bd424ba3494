import sys, numpy as np
sys.path.insert(0, '.')
import oracle
from paper_2406_17284_b200 import ltl
orc = oracle.Oracle()
for n in (32, 64, 128, 256):
    for stats in (False, True):
        rule = ltl.parse_ltl_rule("R1,C2,M0,S2..3,B3..3,NM")
        init = orc.init_random(n, 0.5, 1)
        exp = orc.simulate(init, rule.ints(), 3)
        with ltl.DeviceTorus(n=n) as t:
            t.upload(init)
            try:
                t.run(rule, 3, stats=stats)
                got = t.download()
                print(n, stats, "ok" if np.array_equal(got, exp) else "MISMATCH", flush=True)
            except Exception as e:
                print(n, stats, "ERR", e, flush=True)
                sys.exit(1)
