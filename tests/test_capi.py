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


@pytest.mark.parametrize("text,max_r,msg", [
    ("R17,C2,M0,S2..3,B3..3,NM", 32, None),
    ("R32,C2,M1,S1000..2000,B1000..1500,NM", 32, None),
    ("R32,C2,M0,S0..64,B1..128,NN", 32, None),
    ("R32,C2,M0,S0..4225,B0..0,NM", 32, "exceeds neighborhood capacity 4224"),
    ("R33,C2,M0,S2..3,B3..3,NM", 32, "unsupported rule: radius 33 outside 1..32"),
    ("R20,C2,M0,S2..3,B3..3,NM", 16, "unsupported rule: radius 20 outside 1..16"),
    ("R20,C2,M0,S2..3,B3..3,NM", 20, None),
    ("R1,C2,M0,S2..3,B3..3,NM", 33, "unsupported rule: radius limit 33 outside 1..32"),
])
def test_wide_radius_rule_parse(lib, text, max_r, msg):
    """Extension: ltl_parse_rule_ext accepts radii up to 32 with the same
    grammar and messages; the reference-signature parser still stops at 16."""
    from paper_2406_17284_b200 import ltl
    if msg is None:
        assert ltl.format_ltl_rule(ltl.parse_ltl_rule(text, max_radius=max_r)) == text
        if int(text[1:text.index(",")]) > 16:
            with pytest.raises(ValueError, match="outside 1..16"):
                ltl.parse_ltl_rule(text)
    else:
        with pytest.raises(ValueError, match=re.escape(msg)):
            ltl.parse_ltl_rule(text, max_radius=max_r)


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


@pytest.mark.parametrize("n,f", [(16, 16), (32, 4), (24, 8), (20, 4), (64, 16), (6, 2), (96, 32)])
@pytest.mark.parametrize("layout", [0, 1])
def test_host_fill_halo_matches_reference(lib, ref, orc, n, f, layout):
    """ltl_host_fill_halo (the drop-in's fill_periodic_halo for host grids, any
    f > 0) against the reference's own fill_periodic_halo, via the padded
    grids the reference writes and the oracle's restatement."""
    import ctypes

    import numpy as np
    interior = orc.init_random(n, 0.4, n + f)
    p = n + 2 * f
    rowmajor = np.zeros((p, p), np.uint8)
    rowmajor[f:f + n, f:f + n] = interior
    want = orc.fill_periodic_halo(rowmajor, n, f)
    if layout == 0:
        buf = rowmajor.copy()
    else:  # fragment-contiguous order (grid.hpp:20-25)
        idx = np.array([[((y // f) * (p // f) + x // f) * f * f + (y % f) * f + x % f
                         for x in range(p)] for y in range(p)])
        buf = np.zeros(p * p, np.uint8)
        buf[idx.ravel()] = rowmajor.ravel()
    st = lib.ltl_host_fill_halo(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), n, f, layout)
    assert st == 0
    got = buf if layout == 0 else buf[idx.ravel()].reshape(p, p)
    assert np.array_equal(got.reshape(p, p), want)


def test_host_fill_halo_errors(lib):
    import ctypes

    import numpy as np
    buf = np.zeros(64, np.uint8)
    ptr = buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
    assert lib.ltl_host_fill_halo(ptr, 6, 4, 0) == 1
    assert b"must be a non-negative multiple of f" in lib.ltl_last_error(None)
    assert lib.ltl_host_fill_halo(ptr, 4, 4, 7) == 1
    assert b"layout error" in lib.ltl_last_error(None)


@pytest.mark.parametrize("line,has,msg", [
    ("", 0, "snapshot format error: missing header line"),
    ("CATSNAP", 1, "snapshot format error: malformed header 'CATSNAP'"),
    ("NOTSNAP 1 16 16 rowmajor", 1, "snapshot format error: bad magic 'NOTSNAP'"),
    ("CATSNAP 2 16 16 rowmajor", 1, "snapshot format error: unsupported version 2"),
    ("CATSNAP 1 16 16 diagonal", 1, "snapshot format error: unknown layout 'diagonal'"),
    ("CATSNAP 1 16 16 rowmajor extra", 1, "snapshot format error: trailing tokens in header"),
    ("CATSNAP 1 17 16 rowmajor", 1, "snapshot format error: bad geometry n=17 f=16"),
])
def test_snapshot_parse_header(lib, line, has, msg):
    """ltl_snapshot_parse_header (the header checks the C++ stream reader and
    the device reader share) -- messages of src/snapshot.cpp:39-66."""
    import ctypes
    n, f, lay = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    assert lib.ltl_snapshot_parse_header(line.encode(), has, ctypes.byref(n), ctypes.byref(f),
                                         ctypes.byref(lay)) == 3
    assert lib.ltl_last_error(None).decode() == msg


def test_snapshot_parse_header_ok(lib):
    import ctypes
    n, f, lay = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    assert lib.ltl_snapshot_parse_header(b"CATSNAP 1 64 8 fragment", 1, ctypes.byref(n),
                                         ctypes.byref(f), ctypes.byref(lay)) == 0
    assert (n.value, f.value, lay.value) == (64, 8, 1)
