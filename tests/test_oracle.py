"""Pin the C restatement (oracle/ltl_oracle.c) before trusting it as the checker.

Three anchors, all independent of this repo's product code:
  * the reference's own known-answer tests (values from proj/tests/test_grid.cpp:9-63),
  * golden fixtures produced by the reference library (tests/golden/*.json),
  * the reference library itself where it was built here (oracle/_ref).
"""
import numpy as np
import pytest

from golden_data import load, parse_rule_text, unpack_grid


def test_splitmix_kat_from_reference_tests(orc):
    # proj/tests/test_grid.cpp:9-19
    assert orc.splitmix(0, 4) == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4,
                                  0x06C45D188009454F, 0xF88BB8A8724C81EC]
    assert orc.splitmix(12345, 2) == [0x22118258A9D111A0, 0x346EDCE5F713F8ED]


def test_splitmix_golden(orc):
    for seed, stream in load("kats.json")["splitmix"].items():
        assert orc.splitmix(int(seed), len(stream)) == [int(v) for v in stream]


def test_alive_threshold_edges(orc):
    # proj/tests/test_grid.cpp:21-37
    assert not orc.alive_threshold(0, 0.0)
    assert orc.alive_threshold(2**64 - 1, 1.0)
    assert orc.alive_threshold(2**63 - 1, 0.5) and not orc.alive_threshold(2**63, 0.5)
    assert orc.alive_threshold(0, 2.0**-70) and not orc.alive_threshold(1, 2.0**-70)
    assert orc.alive_threshold(2**62 - 1, 0.25) and not orc.alive_threshold(2**62, 0.25)
    for t in load("kats.json")["thresholds"]:
        assert orc.alive_threshold(int(t["z"]), float.fromhex(t["density"])) == t["alive"]


def test_init_random_first_row_pin(orc):
    # proj/tests/test_grid.cpp:57-63
    g = orc.init_random(16, 0.5, 0)
    assert list(g[0, :4]) == [0, 1, 1, 0]


def test_init_random_golden_grids(orc):
    for e in load("kats.json")["init_grids"]:
        g = orc.init_random(e["n"], e["density"], e["seed"], e["fill_n"])
        assert np.array_equal(g, unpack_grid(e)), e


def test_init_random_errors(orc):
    with pytest.raises(ValueError):
        orc.init_random(64, 1.5, 1)
    with pytest.raises(ValueError):
        orc.init_random(32, 0.5, 1, 33)


def test_anchors(orc):
    """SURVEY §8c anchors (GoL 1024^2 x 100, Bosco, globe, tangy-ramen)."""
    for a in load("anchors.json")["anchors"]:
        init = orc.init_random(a["n"], a["density"], a["seed"])
        assert int(init.sum()) == a["init_alive"]
        assert f"{orc.fnv1a64(init):016x}" == a["init_fnv"]
        out = orc.simulate(init, parse_rule_text(a["rule"]), a["steps"])
        assert int(out.sum()) == a["alive"], a
        assert f"{orc.fnv1a64(out):016x}" == a["fnv"], a


def test_criterion1_sweep(orc):
    """The acceptance criterion-1 shape (proj/tests/acceptance.cpp:69-146) + f=4/8 geometries."""
    cases = load("criterion1.json")["cases"]
    inits = {}
    for c in cases:
        key = (c["n"], c["density"], c["seed"])
        if key not in inits:
            inits[key] = orc.init_random(*key)
        out = orc.simulate(inits[key], parse_rule_text(c["rule"]), c["steps"])
        assert f"{orc.fnv1a64(out):016x}" == c["fnv"], c


def test_center_multiplicity_m0_m1(orc):
    # proj/tests/test_cat_engine.cpp:216-225: M1 S(a+1)..(b+1) == M0 Sa..b for GoL-like rules
    g = orc.init_random(64, 0.4, 9)
    a = orc.simulate(g, [1, 2, 0, 2, 3, 3, 3, 0], 10)
    b = orc.simulate(g, [1, 2, 1, 3, 4, 3, 3, 0], 10)
    assert np.array_equal(a, b)


def test_reductions_match_reference(orc, ref):
    base = ref.init_random(48, 0.4, 7)
    for r in (1, 3, 8, 16):
        for kind in (0, 1):
            rule = [r, 2, 0, 0, 1, 0, 1, kind]
            import oracle
            h_ref, red_ref = ref.reductions(base, oracle.rule_text(rule))
            h, red = orc.reductions(base, rule)
            assert np.array_equal(h, h_ref[16:64, 16:64])
            assert np.array_equal(red, red_ref[16:64, 16:64])


def test_oracle_matches_reference_engines(orc, ref):
    rng = np.random.default_rng(5)
    for r, kind in ((1, 0), (6, 0), (16, 0), (3, 1), (16, 1)):
        g = (rng.random((64, 64)) < 0.3).astype(np.uint8)
        w = 2 * r + 1
        cap = w * w - 1 if kind == 0 else 2 * w - 2
        rule = [r, 2, 1, cap // 5, cap // 2, cap // 4, cap // 3, kind]
        import oracle
        text = oracle.rule_text(rule)
        for engine in ("cat", "base"):
            assert np.array_equal(orc.simulate(g, rule, 5), ref.run_engine(engine, g, text, 5))


def test_fill_periodic_halo(orc):
    n, h = 16, 16
    p = np.zeros((n + 2 * h, n + 2 * h), np.uint8)
    p[h:h + n, h:h + n] = orc.init_random(n, 0.4, 7)
    out = orc.fill_periodic_halo(p, n, h)
    for y in range(n + 2 * h):
        for x in range(n + 2 * h):
            assert out[y, x] == out[h + (y - h) % n, h + (x - h) % n]


def test_wide_radius_fixtures(orc):
    """The wide-radius extension (17 <= r <= 32): the C restatement against
    fixtures from the reference's own brute-force oracle
    (proj/tests/oracle.hpp:50-68 via tests/golden/make_wide.py)."""
    for c in load("wide.json")["cases"]:
        g = orc.simulate(orc.init_random(c["n"], c["density"], c["seed"]), c["ints"], c["steps"])
        assert int(g.sum()) == c["alive"], c["rule"]
        assert f"{orc.fnv1a64(g):016x}" == c["fnv"], c["rule"]


def test_wide_radius_semantic_oracle(orc, ref):
    """Same, live against the reference's semantic oracle on fresh inputs,
    rectangular-free (it is square only) small tori where windows wrap twice."""
    for n, rule in ((32, [17, 2, 0, 300, 700, 350, 600, 0]), (48, [32, 2, 1, 30, 80, 40, 70, 1]),
                    (64, [24, 2, 0, 1200, 2400, 1201, 2400, 0])):
        g = orc.init_random(n, 0.5, 4)
        assert np.array_equal(ref.semantic_steps(g, rule, 3), orc.simulate(g, rule, 3)), rule
