"""Quick device-vs-oracle diagnosis: one generation on small grids, prints the
mismatch pattern (rows/cols) per engine.  Usage: python tools/diag.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2406_17284_b200 import ltl  # noqa: E402

orc = oracle.Oracle()
for n, text in ((128, "R1,C2,M0,S2..3,B3..3,NM"), (256, "R5,C2,M1,S34..58,B34..45,NM"),
                (64, "R2,C2,M0,S2..6,B3..5,NN")):
    rule = ltl.parse_ltl_rule(text)
    init = orc.init_random(n, 0.4, 1)
    exp = orc.simulate(init, rule.ints(), 1)
    for engine in ("stencil", "cat"):
        try:
            got = ltl.run_engine(engine, init, text, 1)
        except Exception as e:  # noqa: BLE001
            print(engine, n, text, "EXC", type(e).__name__, e)
            continue
        bad = np.argwhere(got != exp)
        print(engine, n, text, "mismatches", len(bad), "alive got/exp", int(got.sum()), int(exp.sum()))
        if len(bad):
            print("  rows", np.unique(bad[:, 0])[:20], "cols", np.unique(bad[:, 1])[:20])
            print("  got[0,:16]", got[0, :16], "\n  exp[0,:16]", exp[0, :16])
