"""Regenerate tests/golden/snapshots/ from the UNMODIFIED reference (oracle/_ref).

Run here (the container that has /root/reference):

    make -C oracle && python tests/golden/make_snapshots.py

* *.bin            -- CATSNAP v1 files written by catsim::snapshot_write
                      (src/snapshot.cpp:18-37) for grids made by the reference's
                      own init_random / make_grid, incl. the cases of
                      proj/tests/test_snapshot.cpp:34-86.
* snapshots.json   -- for each .bin: n, f, layout, FNV-1a-64 of the interior;
                      and the malformed inputs of test_snapshot.cpp:88-121 (plus
                      header edge cases) with the exact message
                      catsim::snapshot_read raises for each.
"""
from __future__ import annotations

import base64
import json
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "snapshots")


def fnv(a: np.ndarray) -> str:
    h = 0xCBF29CE484222325
    for b in np.ascontiguousarray(a, np.uint8).tobytes():
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def main() -> None:
    ref = oracle.Reference()
    os.makedirs(HERE, exist_ok=True)
    files = {}

    def emit(name, grid, f, layout):
        path = os.path.join(HERE, name)
        ref.snapshot_write(grid, path, f=f, layout=layout)
        back, f2, lay2 = ref.snapshot_read(path)
        assert np.array_equal(back, grid) and f2 == f and lay2 == layout
        files[name] = {"n": int(grid.shape[0]), "f": f, "layout": layout, "fnv": fnv(grid),
                       "alive": int(grid.sum())}

    one = np.zeros((16, 16), np.uint8)
    one[2, 3] = 1                                    # test_snapshot.cpp:34-46
    emit("one_cell_16.bin", one, 16, 0)
    emit("random_32_fragment.bin", ref.init_random(32, 0.4, 2), 16, 1)   # :58-66
    emit("empty_0.bin", np.zeros((0, 0), np.uint8), 16, 0)                # :68-74
    emit("random_256_f8.bin", ref.init_random(256, 0.5, 7, f=8), 8, 0)
    emit("random_512.bin", ref.init_random(512, 0.21, 1), 16, 0)

    payload = b"\0" * 256
    valid = b"CATSNAP 1 16 16 rowmajor\n" + payload
    bad_byte = bytearray(valid)
    bad_byte[25 + 40] = 2
    bad_in_cut_row = bytearray(valid[:-100])
    bad_in_cut_row[-3] = 5                           # only in the incomplete last row
    cases = {
        "empty": b"",
        "malformed": b"CATSNAP\n" + payload,
        "bad_magic": b"NOTSNAP 1 16 16 rowmajor\n" + payload,
        "bad_version": b"CATSNAP 2 16 16 rowmajor\n" + payload,
        "bad_layout": b"CATSNAP 1 16 16 diagonal\n" + payload,
        "trailing": b"CATSNAP 1 16 16 rowmajor extra\n" + payload,
        "bad_n": b"CATSNAP 1 17 16 rowmajor\n" + payload,
        "bad_f": b"CATSNAP 1 16 0 rowmajor\n" + payload,
        "negative_n": b"CATSNAP 1 -16 16 rowmajor\n" + payload,
        "newline_only": b"\n",
        "no_newline_header": b"CATSNAP 1 0 16 rowmajor",
        "truncated": valid[:-100],
        "bad_byte": bytes(bad_byte),
        "bad_byte_in_cut_row": bytes(bad_in_cut_row),
        "ok_16": valid,
    }
    malformed = {}
    with tempfile.TemporaryDirectory() as td:
        for name, data in cases.items():
            p = os.path.join(td, name)
            with open(p, "wb") as fh:
                fh.write(data)
            try:
                ref.snapshot_read(p)
                err = None
            except Exception as e:  # noqa: BLE001
                err = str(e)
            malformed[name] = {"b64": base64.b64encode(data).decode(), "error": err}
    with open(os.path.join(HERE, "snapshots.json"), "w") as fh:
        json.dump({"files": files, "malformed": malformed}, fh, indent=1, sort_keys=True)
    for k, v in malformed.items():
        print(f"{k:22s} {v['error']}")


if __name__ == "__main__":
    main()
