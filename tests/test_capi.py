"""CPU-side checks of the C-ABI boundary: the library loads without a GPU,
exports every symbol include/ltl_b200.h declares, and its host-only helpers
(rule grammar, presets, VN probe) match the reference's behaviour."""
import os
import re

import pytest

from golden_data import load

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    with open(os.path.join(ROOT, "include", "ltl_b200.h")) as fh:
        text = fh.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ltl_[a-z_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2406_17284_b200 import _build, ltl
    _build.build()
    return ltl.load_library()


def test_exports_every_declared_symbol(lib):
    from paper_2406_17284_b200 import ltl
    declared = _declared_functions()
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in ltl_b200.h but not exported"
    assert sorted(ltl.EXPORTS) == declared


def test_build_info(lib):
    assert b"sm_100a" in lib.ltl_build_info()


def test_presets_match_reference(lib):
    from paper_2406_17284_b200 import ltl
    ours = ltl.ltl_presets()
    theirs = load("kats.json")["presets"]
    assert [(n, r) for n, r, _ in ours] == [(p["name"], p["rule"]) for p in theirs]
    assert [d for _, _, d in ours] == [p["density"] for p in theirs]
    for p in theirs:
        assert ltl.parse_ltl_rule(p["rule"]).ints() == p["ints"]
        assert ltl.format_ltl_rule(ltl.parse_ltl_rule(p["rule"])) == p["rule"]


def test_vn_probe_matches_reference(lib):
    from paper_2406_17284_b200 import ltl
    for r, ints in load("kats.json")["vn_probe"].items():
        assert ltl.von_neumann_probe_rule(int(r)).ints() == ints


@pytest.mark.parametrize("text,msg", [
    ("R1,C2,M0,S2..3,B3..3,NX", "rule parse error: field N"),
    ("X1,C2,M0,S2..3,B3..3,NM", "rule parse error: field R"),
    ("R1,C3,M0,S2..3,B3..3,NM", "unsupported rule: only two-state"),
    ("R17,C2,M0,S2..3,B3..3,NM", "unsupported rule: radius 17 outside 1..16"),
    ("R1,C2,M2,S2..3,B3..3,NM", "rule parse error: field M"),
    ("R1,C2,M0,S3..2,B3..3,NM", "rule parse error: field S"),
    ("R1,C2,M0,S2..3,B3..1,NM", "rule parse error: field B"),
    ("R1,C2,M0,S2..9,B3..3,NM", "exceeds neighborhood capacity 8"),
    ("R1,C2,M1,S2..9,B3..3,NM", None),
    ("R2,C2,M0,S2..3,B3..3,NN", None),
    ("R1,C2,M0,S2..3,B3..3,NM ", "rule parse error: field N"),
])
def test_rule_parse_errors(lib, text, msg):
    from paper_2406_17284_b200 import ltl
    if msg is None:
        assert ltl.format_ltl_rule(ltl.parse_ltl_rule(text)) == text
    else:
        with pytest.raises(ValueError, match=re.escape(msg)):
            ltl.parse_ltl_rule(text)


def test_rule_parse_agrees_with_reference_library(lib, ref):
    """Same accept/reject decision and message as the reference's parser."""
    from paper_2406_17284_b200 import ltl
    cases = ["R1,C2,M0,S2..3,B3..3,NM", "R16,C2,M0,S170..296,B170..300,NM", "R5,C2,M1,S34..58,B34..45,NM",
             "R3,C2,M0,S0..0,B0..0,NN", "R3,C2,M0,S0..13,B0..12,NN", "R3,C2,M0,S0..14,B0..12,NN",
             "R0,C2,M0,S2..3,B3..3,NM", "R1,C2,M0,S-1..3,B3..3,NM", "R1,C2,M0,S..3,B3..3,NM",
             "R1,C2,M0,S2..3,B3..3", "R1,C2,M0,S2.3,B3..3,NM", ""]
    for text in cases:
        try:
            expect = ("ok", ref.parse_rule(text))
        except ValueError as e:
            expect = ("err", str(e))
        try:
            got = ("ok", ltl.parse_ltl_rule(text).ints())
        except ValueError as e:
            got = ("err", str(e))
        assert got == expect, text


def test_no_device_fails_loudly(lib):
    """Without a GPU the device calls raise; there is no CPU fallback."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2406_17284_b200 import ltl
    with pytest.raises(ltl.LtlCudaError):
        ltl.DeviceTorus(n=64)


def test_geometry_errors_before_device(lib):
    from paper_2406_17284_b200 import ltl
    with pytest.raises(ValueError, match="geometry error: n \\(10\\) must be a non-negative multiple of f \\(16\\)"):
        ltl.DeviceTorus(n=10)
    with pytest.raises(ValueError, match="config error: fragment side must be 4, 8, or 16"):
        ltl.DeviceTorus(n=12, f=6)
