"""Fault-injection fixtures from the UNMODIFIED reference (oracle/_ref):
CatConfig.inject_band_fault flips pi2(0,0) of the band fragments
(proj/src/cat_engine.cpp:277); the faulted run either diverges (its grid is
recorded) or trips the negative-count guard (its message is recorded).

    make -C oracle && python tests/golden/make_faults.py
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    ref = oracle.Reference()
    orc = oracle.Oracle()
    presets = ref.presets()
    cases = []
    rules = []
    for r in (1, 2, 5, 8, 16):
        rules.append(("moore-preset", presets[r - 1][1], presets[r - 1][2]))
        rules.append(("vn-probe", oracle.rule_text(ref.von_neumann_probe_rule(r)), 0.25))
    # M1 rules: the centre is not subtracted, so the guard cannot fire and the
    # faulted grid itself is compared
    rules += [("moore-m1", "R5,C2,M1,S34..58,B34..45,NM", 0.21),
              ("moore-m1", "R1,C2,M1,S3..4,B3..3,NM", 0.4),
              ("moore-m1", "R16,C2,M1,S171..297,B170..300,NM", 0.26),
              ("vn-m1", "R3,C2,M1,S4..9,B3..6,NN", 0.3)]
    for kind, rule, dens in rules:
        r = ref.parse_rule(rule)[0]
        for f, sizes in ((16, (32, 64, 128, 256)), (8, (24, 64)), (4, (20, 36))):
            if r > f:
                continue
            for n in sizes:
                for steps in (1, 3):
                    init = ref.init_random(n, dens, 7, f)
                    e = dict(kind=kind, rule=rule, n=n, f=f, density=dens, seed=7, steps=steps)
                    try:
                        out = ref.run_engine("cat", init, rule, steps, f=f, inject_fault=True)
                        e.update(alive=int(out.sum()), fnv=f"{orc.fnv1a64(out):016x}")
                        clean = ref.run_engine("cat", init, rule, steps, f=f)
                        e["diverged"] = bool((clean != out).any())
                    except RuntimeError as ex:
                        e["error"] = str(ex)
                    cases.append(e)
    with open(os.path.join(HERE, "faults.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_faults.py (reference oracle/_ref, cat engine, "
                                "inject_band_fault)", "seed_f": "init_random(n, density, 7, f)",
                   "cases": cases}, fh, indent=0)
    n_err = sum("error" in c for c in cases)
    print(f"{len(cases)} cases, {n_err} guard aborts, "
          f"{sum(c.get('diverged', False) for c in cases)} diverged")


if __name__ == "__main__":
    main()
