"""Generate tests/golden/wide.json: fixtures for the wide-radius extension
(17 <= r <= 32) from the REFERENCE'S OWN brute-force semantic oracle.

    make -C oracle && python tests/golden/make_wide.py

The reference's engines reject r > 16 (proj/src/rule.cpp:33-35), but its
test oracle proj/tests/oracle.hpp:50-68 (torus_rule_steps: explicit modular
wrap, counts re-derived from the rule semantics) takes any LtlRule -- it is
the reference's definition of the LTL step at every radius.  ref_shim.cpp's
ref_semantic_steps runs it unmodified; every number below comes from it, and
each case is also checked against this repo's C restatement (oracle/).

Rules: majority rules at wide radii (the shape of the r = 4 preset
"majority", S40..80 B41..80: survive with at least half, be born with more
than half of the neighbours alive; density 0.5 -- coarsening domains that stay
non-trivial for many generations), Moore and simplified von Neumann, M0 and
M1; Moore rules with the range ratios of the r = 16 preset tangy-ramen
(S 0.156..0.272 N, B 0.156..0.275 N, density 0.26); the reference's VN probe
formula (src/rule.cpp:142-152).
"""
from __future__ import annotations

import concurrent.futures as cf
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def moore_rule(r: int, m: int = 0):
    n = (2 * r + 1) ** 2
    return [r, 2, m, int(0.156 * n), int(0.272 * n), int(0.156 * n), int(0.275 * n), 0]


def majority(r: int, vn: bool = False, m: int = 0):
    cells = 4 * r if vn else (2 * r + 1) ** 2 - 1  # neighbours, centre excluded
    return [r, 2, m, cells // 2 + m, cells + m, cells // 2 + 1, cells, 1 if vn else 0]


def vn_probe(r: int):
    cross = 4 * r + 1  # src/rule.cpp:142-152
    return [r, 2, 0, max(1, cross // 6), cross // 2, max(1, cross // 5), cross // 3, 1]


def rule_text(v) -> str:
    return f"R{v[0]},C{v[1]},M{v[2]},S{v[3]}..{v[4]},B{v[5]}..{v[6]},N{'M' if v[7] == 0 else 'N'}"


def specs():
    out = []
    for r in (17, 18, 20, 23, 24, 27, 28, 31, 32):
        n = 512 if r >= 25 else 256
        out.append((majority(r), n, 0.5, 1, (1, 5)))
    out.append((majority(20, m=1), 256, 0.5, 2, (1, 5)))
    out.append((majority(32, m=1), 512, 0.5, 2, (1, 4)))
    out.append((majority(32), 128, 0.5, 3, (1, 3)))   # window 65 of a 128 torus
    for r in (17, 24, 32):
        out.append((majority(r, vn=True), 256, 0.5, 1, (1, 5)))
    for r in (20, 32):
        out.append((moore_rule(r), 512 if r > 24 else 256, 0.26, 1, (1, 2)))
    for r in (17, 32):
        out.append((vn_probe(r), 256, 0.25, 1, (1, 2)))
    return out


def run(spec):
    rule, n, density, seed, steps = spec
    ref = oracle.Reference()
    orc = oracle.Oracle()
    g = orc.init_random(n, density, seed)
    res = []
    done = 0
    for s in steps:
        g = ref.semantic_steps(g, rule, s - done)
        done = s
        assert np.array_equal(g, orc.simulate(orc.init_random(n, density, seed), rule, s)), (rule, s)
        res.append({"rule": rule_text(rule), "ints": rule, "n": n, "density": density,
                    "seed": seed, "steps": s, "alive": int(g.sum()),
                    "fnv": f"{orc.fnv1a64(g):016x}"})
    return res


def main() -> None:
    cases = []
    with cf.ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:
        for res in ex.map(run, specs()):
            cases.extend(res)
            print(res[-1]["rule"], res[-1]["n"], [c["alive"] for c in res], flush=True)
    doc = {"source": "proj/tests/oracle.hpp torus_rule_steps via oracle/ref_shim.cpp "
                     "ref_semantic_steps (unmodified reference code)",
           "cases": cases}
    with open(os.path.join(HERE, "wide.json"), "w") as fh:
        json.dump(doc, fh, indent=1)


if __name__ == "__main__":
    main()
