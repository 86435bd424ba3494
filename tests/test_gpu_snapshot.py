"""CATSNAP v1 snapshots streamed from / to the device (ltl_snapshot_write /
ltl_snapshot_read) against the reference's snapshot_write / snapshot_read
(src/snapshot.cpp:18-91): byte-identical files, fixtures written by the
reference read back exactly, the reference's error for every malformed
payload, multi-chunk and multi-slab geometries."""
import base64
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "snapshots")
with open(os.path.join(HERE, "snapshots.json")) as _fh:
    GOLD = json.load(_fh)


@pytest.fixture(scope="module")
def ltl():
    from paper_2406_17284_b200 import ltl
    return ltl


def fnv(a: np.ndarray) -> str:
    h = 0xCBF29CE484222325
    for b in np.ascontiguousarray(a, np.uint8).tobytes():
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


@pytest.mark.parametrize("name", sorted(GOLD["files"]))
def test_reference_files_round_trip(ltl, tmp_path, name):
    """read a reference-written file into the device, write it back: same bytes."""
    meta = GOLD["files"][name]
    src = os.path.join(HERE, name)
    with ltl.DeviceTorus(n=meta["n"], f=meta["f"]) as t:
        assert t.snapshot_read(src) == meta["layout"]
        grid = t.download()
        assert grid.shape == (meta["n"], meta["n"]) and fnv(grid) == meta["fnv"]
        out = tmp_path / "back.bin"
        t.snapshot_write(str(out), meta["layout"])
    with open(src, "rb") as a:
        assert out.read_bytes() == a.read()


@pytest.mark.parametrize("n,slabs,layout", [(1024, 1, 0), (1024, 3, 1), (4096, 1, 0),
                                            (8192, 2, 0), (16384, 1, 0)])
def test_write_matches_reference_bytes(ltl, ref, tmp_path, n, slabs, layout):
    """device-side init -> streamed file == the reference's snapshot_write of
    the same grid (16384^2 = 8 chunks of 32 MB)."""
    with ltl.DeviceTorus(n=n, slabs=slabs) as t:
        t.init_random(0.3, 5)
        mine = tmp_path / "mine.bin"
        t.snapshot_write(str(mine), layout)
        grid = t.download()
    theirs = tmp_path / "theirs.bin"
    ref.snapshot_write(grid, str(theirs), layout=layout)
    assert mine.stat().st_size == theirs.stat().st_size
    with open(mine, "rb") as a, open(theirs, "rb") as b:
        while True:
            x, y = a.read(1 << 24), b.read(1 << 24)
            assert x == y
            if not x:
                break


def test_read_after_steps_and_continue(ltl, orc, tmp_path):
    """snapshot mid-run, reload into a fresh context, continue: equals one run."""
    text = "R5,C2,M1,S34..58,B34..45,NM"
    init = orc.init_random(512, 0.21, 3)
    with ltl.DeviceTorus(n=512) as t:
        t.upload(init)
        t.run(text, 7)
        t.snapshot_write(str(tmp_path / "mid.bin"))
        t.run(text, 5)
        want = t.download()
    with ltl.DeviceTorus(n=512, slabs=2) as t:
        assert t.snapshot_read(str(tmp_path / "mid.bin")) == 0
        t.run(text, 5)
        assert np.array_equal(t.download(), want)


@pytest.mark.parametrize("case", sorted(GOLD["malformed"]))
def test_malformed_payloads_raise_the_reference_error(ltl, tmp_path, case):
    spec = GOLD["malformed"][case]
    path = tmp_path / case
    data = base64.b64decode(spec["b64"])
    path.write_bytes(data)
    n = 0 if case == "no_newline_header" else 16
    with ltl.DeviceTorus(n=n) as t:
        if spec["error"] is None:
            assert t.snapshot_read(str(path)) == 0
            return
        with pytest.raises(ltl.LtlRuntimeError) as ei:
            t.snapshot_read(str(path))
        assert str(ei.value) == spec["error"]


def test_geometry_and_config_errors(ltl, tmp_path):
    src = os.path.join(HERE, "random_512.bin")
    with ltl.DeviceTorus(n=256) as t:
        with pytest.raises(ValueError, match="geometry error: snapshot n=512 f=16"):
            t.snapshot_read(src)
    with ltl.DeviceTorus(n=512, f=8) as t:
        with pytest.raises(ValueError, match="geometry error"):
            t.snapshot_read(src)
    with ltl.DeviceTorus(rows=256, cols=512) as t:
        with pytest.raises(ValueError, match="config error: snapshots hold square"):
            t.snapshot_write(str(tmp_path / "x.bin"))
    with ltl.DeviceTorus(n=256) as t:
        with pytest.raises(ValueError, match="layout error"):
            t.snapshot_write(str(tmp_path / "x.bin"), 7)
        with pytest.raises(ltl.LtlRuntimeError, match="cannot open '/no-such-dir/y.bin' for writing"):
            t.snapshot_write("/no-such-dir/y.bin")
