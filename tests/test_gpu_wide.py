"""The wide-radius extension on a B200: the Cat engine with 17 <= r <= 32
(32-row boxes, four pass-2 band chunks; "+16 expansion", a range
the reference's engines reject, proj/src/rule.cpp:33-35).

Parity anchors: tests/golden/wide.json, produced by the reference's own
brute-force semantic oracle (proj/tests/oracle.hpp torus_rule_steps, run
unmodified by tests/golden/make_wide.py), and the C restatement (oracle/,
pinned against those fixtures in tests/test_oracle.py) for rectangular
tori, ring slabs and the large sizes.
"""
import numpy as np
import pytest

from golden_data import load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ltl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2406_17284_b200 import ltl as mod
    return mod


def majority(r, vn=False, m=0):
    cells = 4 * r if vn else (2 * r + 1) ** 2 - 1
    return [r, 2, m, cells // 2 + m, cells + m, cells // 2 + 1, cells, 1 if vn else 0]


@pytest.mark.parametrize("path", ["default", "per_launch"])
def test_wide_fixtures(ltl, orc, monkeypatch, path):
    """Every wide.json case (r = 17..32, Moore / VN, M0 / M1) bit-exact; small
    tori take the multi-generation sweep by default, per_launch forces one
    launch per generation."""
    if path == "per_launch":
        monkeypatch.setenv("LTL_NO_SMALL_PERSIST", "1")
    cases = load("wide.json")["cases"]
    fails = []
    for c in cases:
        init = orc.init_random(c["n"], c["density"], c["seed"])
        with ltl.DeviceTorus(n=c["n"]) as t:
            t.upload(init)
            t.run(c["ints"], c["steps"])
            out = t.download()
        if int(out.sum()) != c["alive"] or f"{orc.fnv1a64(out):016x}" != c["fnv"]:
            fails.append((c["rule"], c["n"], c["steps"], int(out.sum()), c["alive"]))
    assert not fails, fails


@pytest.mark.parametrize("rows,cols", [(32, 128), (96, 256), (160, 384), (288, 128), (416, 256)])
def test_wide_rectangular_tori(ltl, orc, rows, cols):
    """Band geometries: a single 32-row band, last bands of 32..128 rows, one
    strip (the horizontal window wraps inside it), window > torus height."""
    rng = np.random.default_rng(rows + cols)
    init = (rng.random((rows, cols)) < 0.5).astype(np.uint8)
    for rule in (majority(17), majority(25, vn=True), majority(32), majority(32, m=1),
                 majority(29, vn=True, m=1)):
        with ltl.DeviceTorus(rows=rows, cols=cols) as t:
            t.upload(init)
            t.run(rule, 3)
            got = t.download()
        assert np.array_equal(got, orc.simulate(init, rule, 3)), (rows, cols, rule)


@pytest.mark.parametrize("slabs", [2, 4])
def test_wide_ring_slabs(ltl, orc, slabs):
    """In-process ring of row slabs: the 32 rows above / below each slab are
    pulled from the neighbours' buffers by the step's own loads."""
    n = 512
    init = orc.init_random(n, 0.5, 5)
    for rule in (majority(32), majority(21, vn=True)):
        with ltl.DeviceTorus(n=n, slabs=slabs, devices=[0] * slabs) as t:
            t.upload(init)
            t.run(rule, 4)
            got = t.download()
        assert np.array_equal(got, orc.simulate(init, rule, 4)), (slabs, rule)


def test_wide_persistent_ring(ltl, orc, monkeypatch):
    """Multi-generation launches on slabs (self-ring of one slab)."""
    monkeypatch.setenv("LTL_SELF_RING", "1")
    monkeypatch.setenv("LTL_FORCE_PERSIST", "1")
    init = orc.init_random(512, 0.5, 6)
    rule = majority(30)
    with ltl.DeviceTorus(n=512) as t:
        t.upload(init)
        t.run(rule, 5)
        got = t.download()
    assert np.array_equal(got, orc.simulate(init, rule, 5))


def test_wide_stats_bounds(ltl):
    """All-alive torus: H = 2r+1, R = (2r+1)^2 (Moore) / 2(2r+1) (VN) through
    the checked kernel (the acceptance.cpp:245-277 bounds, at r = 32)."""
    n = 256
    full = np.ones((n, n), np.uint8)
    for rule, h, r in ((majority(32), 65, 65 * 65), (majority(32, vn=True), 65, 130),
                       (majority(20), 41, 41 * 41)):
        with ltl.DeviceTorus(n=n) as t:
            t.upload(full)
            st = t.run(rule, 1, stats=True)
        assert (st["max_h"], st["max_r"]) == (h, r), rule


def test_wide_errors(ltl):
    """The extension needs every wrap done by the loads; the reference-named
    parser and the CUDA-core engines keep the reference's r <= 16."""
    with pytest.raises(ValueError, match="r > 16 needs cols % 128 == 0"):
        with ltl.DeviceTorus(rows=256, cols=200) as t:
            t.run(majority(20), 1)
    with pytest.raises(ValueError, match="r > 16 needs"):
        with ltl.DeviceTorus(rows=100, cols=256) as t:
            t.run(majority(20), 1)
    with pytest.raises(ValueError, match="outside 1..16"):
        with ltl.DeviceTorus(n=256) as t:
            t.run(majority(20), 1, engine="pack")
    with pytest.raises(ValueError, match="outside 1..16"):
        ltl.parse_ltl_rule("R20,C2,M0,S840..1680,B841..1680,NM")
    with pytest.raises(ValueError, match="outside 1..32"):
        ltl.parse_ltl_rule("R33,C2,M0,S840..1680,B841..1680,NM", max_radius=32)


@pytest.mark.parametrize("n,steps", [(16384, 3), (32768, 2)])
def test_wide_large(ltl, orc, n, steps):
    """BASELINE sizes (configs[1] / configs[2] tori) at r = 24 / 32 on the
    default paths (persistent sweep at 16384^2, a launch per generation at
    32768^2) against the C restatement."""
    rule = majority(24) if n == 16384 else majority(32, vn=False, m=1)
    with ltl.DeviceTorus(n=n) as t:
        t.init_random(0.5, 11)
        init = t.download()
        t.run(rule, steps)
        got = t.download()
    want = orc.simulate(init, rule, steps)
    assert int(got.sum()) == int(want.sum())
    assert np.array_equal(got, want)
