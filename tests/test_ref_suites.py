"""The REFERENCE's own unit suites (/root/reference/proj/tests/test_*.cpp),
compiled unmodified against this repo's include/catsim/ drop-in headers and
libltl_b200.so (tests/cpp/ref_suites.mk, doctest-compatible harness
tests/cpp/shim/doctest.h), run as shipped: the strongest drop-in check --
code written against the reference's API builds and passes on the B200 path.

The binaries are built where the reference sources exist (this container,
__graft_entry__.build) and travel to the GPU box under build/ref_suites/.
Host-only suites (rule parsing, fragment tiles, bench statistics) run here on
the CPU; every suite runs on the GPU."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "ref_suites")
HOST_SUITES = ("rule", "fragment", "bench", "cost_model")
ALL_SUITES = ("grid", "layout", "rule", "fragment", "cat_engine", "reference", "snapshot",
              "bench", "cost_model")


def _exe(name):
    path = os.path.join(BIN, f"test_{name}")
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (make -f tests/cpp/ref_suites.mk where the reference exists)")
    return path


def _run(path, timeout=1200):
    res = subprocess.run([path], capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    out = res.stdout + res.stderr
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", out)
    assert m, out[-3000:]
    assert res.returncode == 0 and m.group(3) == "0", out[-4000:]
    return int(m.group(1))


@pytest.mark.parametrize("suite", HOST_SUITES)
def test_reference_host_suite(suite):
    assert _run(_exe(suite)) > 0


@pytest.mark.gpu
@pytest.mark.parametrize("suite", ALL_SUITES)
def test_reference_suite_on_gpu(suite):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    assert _run(_exe(suite)) > 0


@pytest.mark.gpu
def test_reference_acceptance_gate():
    """proj/tests/acceptance.cpp unmodified: all seven hard criteria (1536-triple
    engine equivalence cat == base == pack, Table II from the cost model,
    6 MMAs / (2r+1)^2+2 reads, H=33 / R=1089, band assembly, layout
    bijection, determinism matrix)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    path = os.path.join(BIN, "acceptance")
    if not os.path.exists(path):
        pytest.skip("acceptance not built")
    res = subprocess.run([path], capture_output=True, text=True, timeout=1800, cwd=ROOT)
    out = res.stdout + res.stderr
    for k in range(1, 8):
        assert re.search(rf"PASS criterion {k}:", out), out[-4000:]
    assert "all hard criteria passed" in out and res.returncode == 0, out[-4000:]
