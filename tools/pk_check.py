"""4-bit-cell Cat step vs the u8 Cat step (and the reference's hashes via the
oracle at small sizes): bit-exactness over rules / sizes / paths, then timing.
Run on the GPU box from the repo root: python tools/pk_check.py"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2406_17284_b200 import ltl  # noqa: E402

RULES = ["R1,C2,M0,S2..3,B3..3,NM", "R5,C2,M1,S34..58,B34..45,NM", "R16,C2,M0,S170..296,B170..300,NM",
         "R9,C2,M0,S5..18,B7..12,NN", "R3,C2,M1,S1..4,B2..3,NN", "R8,C2,M0,S100..200,B80..150,NM"]


def run(engine, init, rule, steps, **kw):
    n_r, n_c = init.shape
    with ltl.DeviceTorus(rows=n_r, cols=n_c) as t:
        t.upload(init)
        st = t.run(rule, steps, engine=engine, **kw)
        return t.download(), st


def main():
    bad = 0
    rng = np.random.default_rng(5)
    for (rows, cols) in [(128, 128), (256, 384), (1024, 1024), (4096, 4096), (16384, 16384)]:
        init = (rng.random((rows, cols)) < 0.3).astype(np.uint8)
        for rule in RULES:
            for steps in ([1, 2, 7] if rows <= 4096 else [1, 3]):
                a, sa = run("cat-4bit", init, rule, steps, stats=True)
                b, sb = run("cat", init, rule, steps, stats=True)
                same = np.array_equal(a, b) and sa["max_h"] == sb["max_h"] and sa["max_r"] == sb["max_r"]
                if not same:
                    bad += 1
                    diff = np.argwhere(a != b)
                    print(f"MISMATCH {rows}x{cols} {rule} steps={steps} ndiff={len(diff)} first={diff[:4].tolist()} "
                          f"stats {sa} vs {sb}", flush=True)
        print(f"{rows}x{cols} done, mismatches so far {bad}", flush=True)
    # fault injection: same faulted grids / same abort message
    init = (rng.random((1024, 1024)) < 0.3).astype(np.uint8)
    for rule in RULES[:3]:
        outs = []
        for eng in ("cat-4bit", "cat"):
            try:
                outs.append(run(eng, init, rule, 2, inject_fault=True)[0])
            except Exception as e:  # noqa: BLE001
                outs.append(str(e))
        ok = (isinstance(outs[0], str) and outs[0] == outs[1]) or (
            not isinstance(outs[0], str) and not isinstance(outs[1], str) and np.array_equal(outs[0], outs[1]))
        print("fault", rule, "same" if ok else f"DIFFERENT {outs[0] if isinstance(outs[0], str) else ''}"
              f" / {outs[1] if isinstance(outs[1], str) else ''}")
        bad += not ok
    # timing (device, ltl_time)
    for n in (16384, 32768):
        for rule in (RULES[0], RULES[1], RULES[2]):
            for eng in ("cat", "cat-4bit"):
                with ltl.DeviceTorus(n=n) as t:
                    t.init_random(0.3, 1)
                    tot, ker = t.time(rule, 20, warmup=5, engine=eng)
                    print(f"time n={n} {rule[:3]} {eng:8s} {tot / 20 * 1e3:8.1f} us/gen  "
                          f"{n * n * 20 / (tot * 1e-3):.3e} cell updates/s", flush=True)
    print("TOTAL MISMATCHES", bad)


if __name__ == "__main__":
    main()
