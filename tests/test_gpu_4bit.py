"""The Cat step on 4-bit device cells (engine "cat-4bit", LTL_FLAG_4BIT_CELLS;
SURVEY §8f rank 3): two cells per byte in HBM, pass 1 on tcgen05.mma
kind::f8f6f4 (e4m3 band weights x e2m1 cells, f16 accumulators), converted
from / back to the u8 slab around every call.  It must give the reference's
bytes wherever it runs -- the BASELINE configs at their stated sizes against
the reference-generated fixtures, the oracle on small tori (per launch and
persistent), the reference's faulted runs, the H / R bounds -- and it must
actually run (pack / unpack launches counted)."""
import numpy as np
import pytest

from golden_data import load, parse_rule_text
from test_gpu_large import _entries, _series

pytestmark = pytest.mark.gpu

ENGINE = "cat-4bit"


@pytest.fixture(scope="module")
def ltl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2406_17284_b200 import ltl as mod
    return mod


def test_4bit_path_taken(ltl):
    """An eligible torus runs pack + step + unpack (3 launches for one
    generation); an ineligible one (cols % 128 != 0) silently keeps u8 cells."""
    with ltl.DeviceTorus(rows=256, cols=256) as t:
        t.init_random(0.3, 1)
        l0 = t.kernel_launches()
        t.run("R1,C2,M0,S2..3,B3..3,NM", 1, engine=ENGINE)
        assert t.kernel_launches() - l0 == 3
        l0 = t.kernel_launches()
        t.run("R1,C2,M0,S2..3,B3..3,NM", 1)
        assert t.kernel_launches() - l0 == 1
    with ltl.DeviceTorus(rows=256, cols=200) as t:
        t.init_random(0.3, 1)
        l0 = t.kernel_launches()
        t.run("R1,C2,M0,S2..3,B3..3,NM", 1, engine=ENGINE)
        assert t.kernel_launches() - l0 < 3


def test_config1_4bit_16384_1000_generations(ltl, orc):
    es = _entries("c1")
    _series(ltl, orc, es, es[0]["rule"], engine=ENGINE)


def test_config2_4bit_radius_sweep_32768(ltl, orc):
    es = _entries("c2")
    for rule in dict.fromkeys(e["rule"] for e in es):
        _series(ltl, orc, es, rule, engine=ENGINE)


def test_config4_4bit_r8_65536(ltl, orc):
    es = _entries("c4")
    _series(ltl, orc, es, es[0]["rule"], engine=ENGINE)


@pytest.mark.parametrize("persist", ["0", "1"])
@pytest.mark.parametrize("rows,cols", [(128, 128), (256, 384), (1024, 1024), (512, 384)])
def test_4bit_against_oracle(ltl, orc, rows, cols, persist, monkeypatch):
    """Moore and VN at small / middle / large radius, odd and even generation
    counts, one launch per generation and the persistent sweep (forced)."""
    monkeypatch.setenv("LTL_FORCE_PERSIST" if persist == "1" else "LTL_NO_PERSIST", "1")
    rng = np.random.default_rng(rows * 13 + cols)
    init = (rng.random((rows, cols)) < 0.3).astype(np.uint8)
    for text in ("R1,C2,M0,S2..3,B3..3,NM", "R5,C2,M1,S34..58,B34..45,NM",
                 "R16,C2,M0,S170..296,B170..300,NM", "R9,C2,M0,S5..18,B7..12,NN",
                 "R16,C2,M1,S10..40,B20..30,NN"):
        rule = parse_rule_text(text)
        with ltl.DeviceTorus(rows=rows, cols=cols) as t:
            t.upload(init)
            t.run(text, 3, engine=ENGINE)
            assert np.array_equal(t.download(), orc.simulate(init, rule, 3)), (text, 3)
            t.run(text, 4, engine=ENGINE)
            assert np.array_equal(t.download(), orc.simulate(init, rule, 7)), (text, 7)


def test_4bit_fault_injection_matches_reference(ltl, orc):
    """The reference's faulted runs (tests/golden/faults.json) on the tori the
    4-bit path takes (n % 128 == 0): same diverged grid or same abort message."""
    bad, ran = [], 0
    for c in load("faults.json")["cases"]:
        if c["n"] % 128:
            continue
        ran += 1
        init = orc.init_random(c["n"], c["density"], c["seed"])
        with ltl.DeviceTorus(n=c["n"], f=c["f"]) as t:
            t.upload(init)
            try:
                t.run(c["rule"], c["steps"], inject_fault=True, engine=ENGINE)
                out = t.download()
                got = dict(alive=int(out.sum()), fnv=f"{orc.fnv1a64(out):016x}")
            except ltl.LtlLogicError as e:
                got = dict(error=str(e))
        want = {k: c[k] for k in ("alive", "fnv", "error") if k in c}
        if got != want:
            bad.append((c["rule"], c["n"], c["f"], c["steps"], want, got))
    assert ran > 0
    assert not bad, f"{len(bad)} mismatches, first: {bad[:3]}"


def test_4bit_stats_bounds(ltl):
    """acceptance.cpp:245-277: H = 33 and R = 1089 on an all-alive r = 16 torus."""
    with ltl.DeviceTorus(rows=256, cols=256) as t:
        t.upload(np.ones((256, 256), np.uint8))
        st = t.run("R16,C2,M0,S170..296,B170..300,NM", 1, stats=True, engine=ENGINE)
    assert (st["max_h"], st["max_r"]) == (33, 1089)


def test_4bit_time_keeps_u8_current(ltl, orc):
    """ltl_time keeps the 4-bit copy across its generations and brings the u8
    slab up to date before returning: warm-up + timed + sampled generations."""
    text = "R5,C2,M1,S34..58,B34..45,NM"
    init = orc.init_random(1024, 0.21, 3)
    with ltl.DeviceTorus(n=1024) as t:
        t.upload(init)
        t.time(text, 4, warmup=3, engine=ENGINE)
        got = t.download()
    # warm-up 3 + timed 4 + the per-launch kernel-time sample (4, persistent: 0)
    ok = any(np.array_equal(got, orc.simulate(init, parse_rule_text(text), k)) for k in (7, 11))
    assert ok
