"""Small runs of every device kernel for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python tools/sanitize.py

Each case is checked against the C oracle too, so a sanitizer run is also a
parity run.  Kept small: the sanitizers slow kernels down 10-100x."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
from golden_data import parse_rule_text  # noqa: E402
from paper_2406_17284_b200 import ltl  # noqa: E402


def main():
    orc = oracle.Oracle()
    cases = [("R1,C2,M0,S2..3,B3..3,NM", 256, 256), ("R16,C2,M0,S170..296,B170..300,NM", 256, 384),
             ("R7,C2,M0,S5..15,B4..10,NN", 200, 136)]
    for text, rows, cols in cases:
        rule = parse_rule_text(text)
        init = (np.random.default_rng(rows + cols).random((rows, cols)) < 0.3).astype(np.uint8)
        want = orc.simulate(init, rule, 3)
        for engine in ("cat", "base", "pack", "cat-4bit"):
            with ltl.DeviceTorus(rows=rows, cols=cols) as t:
                t.upload(init)
                t.run(text, 3, engine=engine, stats=True)
                assert np.array_equal(t.download(), want), (text, engine)
        os.environ["LTL_FORCE_PERSIST"] = "1"  # the multi-generation sweep
        with ltl.DeviceTorus(rows=rows, cols=cols) as t:
            t.upload(init)
            t.run(text, 3)
            assert np.array_equal(t.download(), want), (text, "persistent")
        del os.environ["LTL_FORCE_PERSIST"]
        print("ok", text, rows, cols, flush=True)
    with ltl.DeviceTorus(n=128, slabs=2, devices=[0, 0]) as t:  # ring of slabs
        t.init_random(0.3, 1)
        g = t.download()
        t.run("R5,C2,M1,S34..58,B34..45,NM", 2)
        assert np.array_equal(t.download(), orc.simulate(g, parse_rule_text("R5,C2,M1,S34..58,B34..45,NM"), 2))
    with ltl.DeviceTorus(n=64, f=8) as t:  # padded fragment-layout transfers
        t.init_random(0.4, 2)
        p = t.download_padded(ltl.LAYOUT_FRAGMENT)
        t.upload_padded(p, ltl.LAYOUT_FRAGMENT)
    os.environ["LTL_TC_GRID"] = "3"  # 8 bands >= 3 CTAs: the dynamic remainder schedule
    os.environ["LTL_NO_PERSIST"] = "1"
    g = (np.random.default_rng(5).random((1024, 512)) < 0.3).astype(np.uint8)
    with ltl.DeviceTorus(rows=1024, cols=512) as t:
        t.upload(g)
        t.run("R5,C2,M1,S34..58,B34..45,NM", 3)
        assert np.array_equal(t.download(), orc.simulate(g, parse_rule_text("R5,C2,M1,S34..58,B34..45,NM"), 3))
    del os.environ["LTL_TC_GRID"], os.environ["LTL_NO_PERSIST"]
    with ltl.DeviceTorus(n=2048) as t:  # bit-packed host <-> device transfers (>= 4 MB)
        g = (np.random.default_rng(9).random((2048, 2048)) < 0.3).astype(np.uint8)
        t.upload(g)
        assert np.array_equal(t.download(), g)
        t.run("R1,C2,M0,S2..3,B3..3,NM", 1, engine="cat-4bit")
        assert np.array_equal(t.download(), orc.simulate(g, parse_rule_text("R1,C2,M0,S2..3,B3..3,NM"), 1))
    print("sanitize cases done")


if __name__ == "__main__":
    main()
