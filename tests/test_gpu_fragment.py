"""The reference's fragment-level passes (horizontal_step, vertical_step_moore,
vertical_step_von_neumann; src/cat_engine.cpp:123-258) materialised on the
device (ltl_fragment_pass) against the UNMODIFIED reference (oracle/_ref):
identical padded H and R fields, halo fragments included."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def frag_order(n, f):
    """Row-major padded index of every fragment-contiguous position."""
    p = n + 2 * f
    fpr = p // f
    idx = np.empty(p * p, np.int64)
    k = 0
    for fi in range(fpr):
        for fj in range(fpr):
            for a in range(f):
                for c in range(f):
                    idx[k] = (fi * f + a) * p + fj * f + c
                    k += 1
    return idx


def bands(f, r):
    a = np.arange(f)[:, None]
    b = np.arange(f)[None, :]
    pi1 = (a - b >= f - r).astype(np.int32)
    pi2 = (np.abs(a - b) <= r).astype(np.int32)
    pi3 = (b - a >= f - r).astype(np.int32)
    return np.concatenate([pi1.ravel(), pi2.ravel(), pi3.ravel()])


def run_pass(lib, stage, n, f, cells_frag, bw, h_frag=None):
    out = np.zeros(cells_frag.size, np.int32)
    P = ctypes.POINTER
    st = lib.ltl_fragment_pass(
        stage, n, f, cells_frag.ctypes.data_as(P(ctypes.c_uint8)),
        bw.ctypes.data_as(P(ctypes.c_int32)),
        h_frag.ctypes.data_as(P(ctypes.c_int32)) if h_frag is not None else None,
        out.ctypes.data_as(P(ctypes.c_int32)))
    assert st == 0, lib.ltl_last_error(None).decode()
    return out


@pytest.mark.parametrize("n,f", [(48, 16), (32, 8), (20, 4)])
def test_fragment_passes_match_reference(ref, n, f):
    from paper_2406_17284_b200 import ltl
    lib = ltl.load_library()
    order = frag_order(n, f)
    rng = np.random.default_rng(n + f)
    grid = (rng.random((n, n)) < 0.4).astype(np.uint8)
    padded = np.pad(grid, f, mode="wrap")  # fill_periodic_halo (f <= n here)
    cells = np.ascontiguousarray(padded.ravel()[order])
    for r in sorted({1, 2, f // 2, f}):
        for kind in ("NM", "NN"):
            text = (f"R{r},C2,M0,S1..2,B1..2,{kind}" if kind == "NN"
                    else f"R{r},C2,M0,S1..2,B1..2,NM")
            h_ref, r_ref = ref.reductions(grid, text, f)
            bw = bands(f, r)
            h = run_pass(lib, 0, n, f, cells, bw)
            red = run_pass(lib, 1 if kind == "NM" else 2, n, f, cells, bw, h)
            h_rm = np.empty_like(h)
            h_rm[order] = h
            r_rm = np.empty_like(red)
            r_rm[order] = red
            assert np.array_equal(h_rm, h_ref.ravel()), (n, f, r, kind, "H")
            assert np.array_equal(r_rm, r_ref.ravel()), (n, f, r, kind, "R")
