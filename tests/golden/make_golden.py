"""Regenerate tests/golden/*.json from the UNMODIFIED reference (oracle/_ref).

Run here (the container that has /root/reference):

    make -C oracle && python tests/golden/make_golden.py

Every number in the fixtures is produced by the reference library itself
(run_engine through ref_shim.cpp), never by this repo's code:

* anchors.json    -- the SURVEY.md §8c / BASELINE.md §4 parity anchors: rule,
                     n, density, seed, steps -> alive count and FNV-1a-64 of the
                     row-major interior, for both the `cat` and `base` engines.
* criterion1.json -- the acceptance criterion-1 sweep shape
                     (proj/tests/acceptance.cpp:69-146): r = 1..16 x {Moore preset,
                     VN probe} x n in {32, 64, 128} x seeds 1..8 x steps {1, 25},
                     plus f = 4 / 8 geometries with n not a multiple of 16.
* kats.json       -- splitmix64 streams, alive_threshold edges, presets, the VN
                     probe rules and small init_random grids.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def fnv(a: np.ndarray) -> str:
    h = 0xCBF29CE484222325
    for b in np.ascontiguousarray(a, np.uint8).tobytes():
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def fnv_fast(ref_oracle: oracle.Oracle, a: np.ndarray) -> str:
    return f"{ref_oracle.fnv1a64(a):016x}"


def main() -> None:
    ref = oracle.Reference()
    orc = oracle.Oracle()
    workers = max(1, ref.hardware_concurrency())
    presets = ref.presets()

    # --- anchors -----------------------------------------------------------
    anchor_specs = [
        ("R1,C2,M0,S2..3,B3..3,NM", 1024, 0.5, 1, 100),
        ("R5,C2,M1,S34..58,B34..45,NM", 1024, 0.21, 1, 100),
        ("R5,C2,M1,S34..58,B34..45,NM", 1024, 0.5, 1, 100),
        ("R5,C2,M0,S35..59,B34..45,NM", 1024, 0.21, 1, 100),
        ("R5,C2,M0,S35..59,B34..45,NM", 2048, 0.21, 1, 10),
        ("R8,C2,M0,S163..223,B74..252,NM", 1024, 0.23, 1, 25),
        ("R16,C2,M0,S170..296,B170..300,NM", 1024, 0.26, 1, 25),
        ("R16,C2,M0,S170..296,B170..300,NM", 2048, 0.26, 1, 10),
    ]
    anchors = []
    for rule, n, dens, seed, steps in anchor_specs:
        t0 = time.time()
        init = ref.init_random(n, dens, seed)
        out_cat = ref.run_engine("cat", init, rule, steps, workers=workers)
        entry = dict(rule=rule, n=n, density=dens, seed=seed, steps=steps,
                     init_alive=int(init.sum()), init_fnv=fnv_fast(orc, init),
                     alive=int(out_cat.sum()), fnv=fnv_fast(orc, out_cat), engines=["cat"])
        if n <= 1024:
            out_base = ref.run_engine("base", init, rule, steps)
            assert np.array_equal(out_base, out_cat), rule
            entry["engines"].append("base")
        anchors.append(entry)
        print(f"anchor {rule} n={n} -> alive {entry['alive']} {entry['fnv']} "
              f"({time.time() - t0:.1f}s)", flush=True)
    with open(os.path.join(HERE, "anchors.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py (reference oracle/_ref)",
                   "hash": "FNV-1a-64 over the n*n row-major interior bytes",
                   "anchors": anchors}, fh, indent=1)

    # --- criterion-1 sweep -------------------------------------------------
    cases = []
    for r in range(1, 17):
        moore_rule, moore_density = presets[r - 1][1], presets[r - 1][2]
        vn_rule = oracle.rule_text(ref.von_neumann_probe_rule(r))
        for kind, rule, dens in (("moore", moore_rule, moore_density), ("vn", vn_rule, 0.25)):
            for n in (32, 64, 128):
                for seed in range(1, 9):
                    init = ref.init_random(n, dens, seed)
                    for steps in (1, 25):
                        out, st = ref.run_engine("cat", init, rule, steps, stats=True)
                        cases.append(dict(r=r, kind=kind, rule=rule, n=n, f=16, density=dens,
                                          seed=seed, steps=steps, alive=int(out.sum()),
                                          fnv=fnv_fast(orc, out), max_h=st["max_h"],
                                          max_r=st["max_r"], mma_count=st["mma_count"]))
    # small / non-16 geometries (f = 4, 8) and the 2r+1 > n wrap cases (n = 16)
    for f, n_list in ((4, (4, 8, 20, 36)), (8, (8, 24, 40)), (16, (16,))):
        for r in range(1, f + 1):
            moore_rule, dens = presets[r - 1][1], presets[r - 1][2]
            vn_rule = oracle.rule_text(ref.von_neumann_probe_rule(r))
            for kind, rule, d in (("moore", moore_rule, dens), ("vn", vn_rule, 0.25)):
                for n in n_list:
                    for seed in (1, 2):
                        init = ref.init_random(n, d, seed, f)
                        for steps in (1, 7):
                            out, st = ref.run_engine("cat", init, rule, steps, f=f, stats=True)
                            cases.append(dict(r=r, kind=kind, rule=rule, n=n, f=f, density=d,
                                              seed=seed, steps=steps, alive=int(out.sum()),
                                              fnv=fnv_fast(orc, out), max_h=st["max_h"],
                                              max_r=st["max_r"], mma_count=st["mma_count"]))
    with open(os.path.join(HERE, "criterion1.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py (reference oracle/_ref, cat engine)",
                   "cases": cases}, fh)
    print(f"criterion1: {len(cases)} cases", flush=True)

    # --- KATs ----------------------------------------------------------------
    thresholds = []
    for z, d in [(0, 0.0), (2**64 - 1, 0.0), (0, 1.0), (2**64 - 1, 1.0), (2**63 - 1, 0.5),
                 (2**63, 0.5), (0, 2.0**-70), (1, 2.0**-70), (0, 2.0**-100), (1, 2.0**-100),
                 (2**62 - 1, 0.25), (2**62, 0.25), (12345678901234567, 0.37),
                 (0x5E2A000000000000, 0.37), (0x5EB851EB851EB851, 0.37),
                 (0x5EB851EB851EB852, 0.37), (0x5EB851EB851EB800, 0.37)]:
        thresholds.append(dict(z=str(z), density=d.hex(), alive=ref.alive_threshold(z, d)))
    grids = []
    for n, d, seed, fill in [(16, 0.5, 0, -1), (32, 0.37, 99, -1), (64, 1.0, 3, 48),
                             (48, 0.35, 42, -1), (20, 0.3, 5, 13)]:
        f = 4 if n == 20 else 16
        g = ref.init_random(n, d, seed, f, fill)
        grids.append(dict(n=n, density=d, seed=seed, f=f, fill_n=fill,
                          bits=np.packbits(g).tobytes().hex()))
    kats = dict(
        splitmix={str(s): [str(v) for v in ref.splitmix(s, 8)] for s in (0, 1, 12345, 2**63 + 7)},
        thresholds=thresholds,
        presets=[dict(name=a, rule=b, density=c, ints=ref.parse_rule(b)) for a, b, c in presets],
        vn_probe={str(r): ref.von_neumann_probe_rule(r) for r in range(1, 17)},
        init_grids=grids,
    )
    with open(os.path.join(HERE, "kats.json"), "w") as fh:
        json.dump(kats, fh, indent=1)
    print("kats written")


if __name__ == "__main__":
    main()
