"""Parity at the sizes BASELINE.json's configs state, against fixtures the
UNMODIFIED reference produced at those sizes (tests/golden/large_c*.json,
generator tests/golden/make_large.py; alive count + FNV-1a-64 of the whole
n x n interior + FNV of 16 row blocks):

  configs[1]  Bosco r=5 (R5,C2,M1,S34..58,B34..45,NM) 16384^2, generations
              1 / 10 / 100 / 1000 -- the DEFAULT path (the persistent
              multi-generation sweep at this size), as bench configs[1] runs it;
  configs[2]  every Table III preset r=1..16 at 32768^2, generations 1 and 2
              (one launch per generation, the bench's headline path);
  configs[3]  r=16 tangy-ramen at 65536^2 (a 4.3 GB slab: byte offsets past
              2^31), generations 1 and 2, one slab and the 2/4/8-slab strong-
              scaling partition (virtual slabs on one GPU, rows exchanged
              between slabs every generation);
  configs[4]  r=8 globe at 65536^2 (the weak-scaling per-GPU torus), 1 and 2.

The initial grids are made on the device (ltl_init_random) and are checked
against the reference's init_random digest first."""
import os

import numpy as np
import pytest

from golden_data import GOLDEN, load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ltl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2406_17284_b200 import ltl as mod
    return mod


def _entries(cfg):
    path = os.path.join(GOLDEN, f"large_{cfg}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated yet")
    return load(f"large_{cfg}.json")["entries"]


def _digest_ok(orc, grid, e):
    """(ok, detail): full-grid alive + FNV, and the first differing row block."""
    alive = int(np.count_nonzero(grid))
    fnv = f"{orc.fnv1a64(grid):016x}"
    if alive == e["alive"] and fnv == e["fnv"]:
        return True, ""
    rb = e["block_rows"]
    bad = [i for i in range(16) if f"{orc.fnv1a64(grid[i * rb:(i + 1) * rb]):016x}" != e["block_fnv"][i]]
    return False, f"alive {alive} vs {e['alive']}, differing row blocks {bad}"


def _series(ltl, orc, entries, rule, slabs=1, engine="cat"):
    """Device init + the fixture's generation checkpoints on one torus."""
    es = sorted((e for e in entries if e["rule"] == rule), key=lambda e: e["steps"])
    assert es and es[0]["steps"] == 0, rule
    n, dens = es[0]["n"], es[0]["density"]
    kw = dict(n=n, slabs=slabs, devices=[0] * slabs) if slabs > 1 else dict(rows=n, cols=n)
    with ltl.DeviceTorus(**kw) as t:
        t.init_random(dens, es[0]["seed"])
        done = 0
        for e in es:
            if e["steps"] > done:
                t.run(rule, e["steps"] - done, engine=engine)
                done = e["steps"]
            ok, why = _digest_ok(orc, t.download(), e)
            assert ok, f"{rule} n={n} slabs={slabs} {engine} after {done} generations: {why}"


def test_config1_bosco_16384_1000_generations(ltl, orc):
    es = _entries("c1")
    _series(ltl, orc, es, es[0]["rule"])


def test_config2_radius_sweep_32768(ltl, orc):
    es = _entries("c2")
    for rule in dict.fromkeys(e["rule"] for e in es):
        _series(ltl, orc, es, rule)


@pytest.mark.parametrize("engine", ["pack"])
def test_config2_radius_sweep_32768_stencil(ltl, orc, engine):
    """The CUDA-core packed stencil at the same size, a few radii."""
    es = _entries("c2")
    rules = list(dict.fromkeys(e["rule"] for e in es))
    for rule in rules[::5]:
        _series(ltl, orc, [e for e in es if e["steps"] <= 1], rule, engine=engine)


@pytest.mark.parametrize("slabs", [1, 2, 4, 8])
def test_config3_r16_65536(ltl, orc, slabs):
    es = _entries("c3")
    _series(ltl, orc, es, es[0]["rule"], slabs=slabs)


def test_config4_r8_65536(ltl, orc):
    es = _entries("c4")
    _series(ltl, orc, es, es[0]["rule"])
