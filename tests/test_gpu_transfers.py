"""Bit-packed host <-> device transfers (csrc/host/xfer_bits.cpp + the device
expand / pack kernels): every upload / download of >= 4 MB of rows whose
width is a multiple of 32 crosses PCIe as one bit per cell.  The bytes that
land must be exactly the byte copies' -- pinned and pageable host memory,
dense interiors and padded grids (both layouts), and grids holding bytes that
are not cells (then both directions fall back to byte copies)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ltl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2406_17284_b200 import ltl as mod
    return mod


def _pinned(shape):
    import torch
    return torch.empty(shape, dtype=torch.uint8).pin_memory().numpy()


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("rows,cols", [(4096, 4096), (2048, 2080), (12288, 512)])
def test_interior_roundtrip(ltl, rows, cols, pinned):
    rng = np.random.default_rng(rows + cols)
    g = (rng.random((rows, cols)) < 0.4).astype(np.uint8)
    src = _pinned(g.shape) if pinned else np.empty_like(g)
    src[...] = g
    dst = _pinned(g.shape) if pinned else np.empty_like(g)
    with ltl.DeviceTorus(rows=rows, cols=cols) as t:
        t.upload(src)
        t.download(dst)
    assert np.array_equal(dst, g)


def test_non_cell_bytes_fall_back(ltl):
    """Bytes other than 0 / 1 are not cells; they must survive an upload /
    download round trip exactly as with byte copies."""
    rng = np.random.default_rng(3)
    g = (rng.random((4096, 4096)) < 0.4).astype(np.uint8)
    g[17, 33] = 2
    g[4000, 4095] = 255
    with ltl.DeviceTorus(rows=4096, cols=4096) as t:
        t.upload(g)
        assert np.array_equal(t.download(), g)


@pytest.mark.parametrize("layout", [0, 1])
def test_padded_roundtrip_and_run(ltl, orc, layout):
    """ltl_upload / ltl_download of a padded (n + 2f)^2 host grid (the C++
    drop-in's path), then a run: equal to the byte-copy path
    (LTL_BYTE_TRANSFERS) and to the oracle."""
    import os
    n, f = 2048, 16
    init = orc.init_random(n, 0.3, 5)
    outs = []
    for env in (None, "1"):
        if env:
            os.environ["LTL_BYTE_TRANSFERS"] = env
        try:
            with ltl.DeviceTorus(n=n, f=f) as t:
                t.upload(init)
                t.run("R5,C2,M1,S34..58,B34..45,NM", 3)
                outs.append(t.download())
                padded = t.download_padded(layout)
                t.upload_padded(padded, layout)
                outs.append(t.download())
        finally:
            os.environ.pop("LTL_BYTE_TRANSFERS", None)
    ref = orc.simulate(init, __import__("golden_data").parse_rule_text("R5,C2,M1,S34..58,B34..45,NM"), 3)
    for o in outs:
        assert np.array_equal(o, ref)


def test_run_interior_bits_equal_bytes(ltl, orc):
    """ltl_run_interior (run_engine(Cat), the bench's e2e call) with and without
    the bit-packed transfers."""
    import os
    n = 4096
    g = orc.init_random(n, 0.21, 1)
    hin, hout = _pinned((n, n)), _pinned((n, n))
    hin[...] = g
    res = []
    for env in (None, "1"):
        if env:
            os.environ["LTL_BYTE_TRANSFERS"] = env
        try:
            with ltl.DeviceTorus(n=n) as t:
                t.run_interior(hin, "R5,C2,M1,S34..58,B34..45,NM", 4, out=hout)
                res.append(hout.copy())
        finally:
            os.environ.pop("LTL_BYTE_TRANSFERS", None)
    assert np.array_equal(res[0], res[1])
