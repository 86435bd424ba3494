"""CATSNAP v1 header logic on the host (no device): ltl_snapshot_probe against
the reference's snapshot_read (src/snapshot.cpp:39-66) through the fixtures of
tests/golden/snapshots/ (made by make_snapshots.py from oracle/_ref)."""
import base64
import json
import os

import numpy as np
import pytest

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "snapshots")
with open(os.path.join(HERE, "snapshots.json")) as _fh:
    GOLD = json.load(_fh)

# payload-level failures: the header is fine, so the probe accepts it
PAYLOAD_CASES = {"truncated", "bad_byte", "bad_byte_in_cut_row", "ok_16", "no_newline_header"}


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
def test_fixture_files_parse(ltl, name):
    meta = GOLD["files"][name]
    path = os.path.join(HERE, name)
    assert ltl.snapshot_probe(path) == (meta["n"], meta["f"], meta["layout"])
    with open(path, "rb") as fh:
        data = fh.read()
    header = data[:data.index(b"\n") + 1]
    token = b"rowmajor" if meta["layout"] == 0 else b"fragment"
    assert header == b"CATSNAP 1 %d %d %s\n" % (meta["n"], meta["f"], token)
    body = np.frombuffer(data[len(header):], np.uint8)
    assert body.size == meta["n"] ** 2 and fnv(body) == meta["fnv"]


@pytest.mark.parametrize("name", sorted(GOLD["files"]))
def test_fixtures_pinned_to_reference(ref, name):
    meta = GOLD["files"][name]
    grid, f, layout = ref.snapshot_read(os.path.join(HERE, name))
    assert (grid.shape[0], f, layout) == (meta["n"], meta["f"], meta["layout"])
    assert fnv(grid) == meta["fnv"]


@pytest.mark.parametrize("case", sorted(GOLD["malformed"]))
def test_header_errors_match_reference(ltl, tmp_path, case):
    spec = GOLD["malformed"][case]
    path = tmp_path / case
    path.write_bytes(base64.b64decode(spec["b64"]))
    if case in PAYLOAD_CASES:
        n, f, layout = ltl.snapshot_probe(str(path))
        assert f == 16 and layout == 0 and n in (0, 16)
        return
    with pytest.raises(ltl.LtlRuntimeError) as ei:
        ltl.snapshot_probe(str(path))
    assert str(ei.value) == spec["error"]


def test_malformed_messages_pinned_to_reference(ref, tmp_path):
    for case, spec in GOLD["malformed"].items():
        path = tmp_path / case
        path.write_bytes(base64.b64decode(spec["b64"]))
        try:
            ref.snapshot_read(str(path))
            err = None
        except Exception as e:  # noqa: BLE001
            err = str(e)
        assert err == spec["error"], case


def test_cannot_open(ltl, ref):
    path = "/no-such-dir/x.bin"
    with pytest.raises(ltl.LtlRuntimeError) as ei:
        ltl.snapshot_probe(path)
    with pytest.raises(Exception) as er:
        ref.snapshot_read(path)
    assert str(ei.value) == str(er.value) == f"snapshot format error: cannot open '{path}' for reading"
