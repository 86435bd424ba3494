"""Loader for the committed reference-generated fixtures in tests/golden/."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name: str):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def unpack_grid(entry) -> np.ndarray:
    n = entry["n"]
    bits = np.frombuffer(bytes.fromhex(entry["bits"]), np.uint8)
    return np.unpackbits(bits)[: n * n].reshape(n, n)


def parse_rule_text(text: str):
    """Minimal parser for fixture rule strings (grammar of src/rule.cpp:61-87)."""
    parts = dict((p[0], p[1:]) for p in text.split(","))
    s1, s2 = (int(v) for v in parts["S"].split(".."))
    b1, b2 = (int(v) for v in parts["B"].split(".."))
    return [int(parts["R"]), int(parts["C"]), int(parts["M"]), s1, s2, b1, b2,
            0 if parts["N"] == "M" else 1]
