"""Parity of the device engines with the reference, on a B200.

Every grid the CUDA path produces is compared byte-for-byte with the C
restatement of the reference (oracle/, pinned in tests/test_oracle.py) and/or
the reference-generated golden fixtures (tests/golden/).  Both engines are
exercised through the C-ABI: "cat" (tcgen05 banded MMA), "base" (the
CUDA-core direct-sum stencil) and "pack" (the CUDA-core packed sliding-window
stencil).
"""
import numpy as np
import pytest

from golden_data import load, parse_rule_text

pytestmark = pytest.mark.gpu

ENGINES = ("cat", "base", "pack")


@pytest.fixture(scope="module")
def ltl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2406_17284_b200 import ltl as mod
    return mod


def _fnv(orc, a):
    return f"{orc.fnv1a64(a):016x}"


@pytest.mark.parametrize("engine", ENGINES)
def test_criterion1_sweep(ltl, orc, engine):
    """acceptance.cpp:69-146 shape: r=1..16 x {Moore preset, VN probe} x n x seeds x
    steps, plus f=4/8 geometries -- against the reference's own hashes."""
    cases = load("criterion1.json")["cases"]
    tori = {}
    inits = {}
    failures = []
    for c in cases:
        key = (c["n"], c["f"])
        if key not in tori:
            tori[key] = ltl.DeviceTorus(n=c["n"], f=c["f"])
        ikey = (c["n"], c["density"], c["seed"])
        if ikey not in inits:
            inits[ikey] = orc.init_random(*ikey)
        t = tori[key]
        t.upload(inits[ikey])
        st = t.run(c["rule"], c["steps"], engine=engine, stats=(c["seed"] == 1))
        out = t.download()
        if _fnv(orc, out) != c["fnv"]:
            failures.append((c["rule"], c["n"], c["f"], c["seed"], c["steps"]))
        elif st is not None and c["f"] == 16 and c["n"] >= 32:
            assert (st["max_h"], st["max_r"]) == (c["max_h"], c["max_r"]), c
    for t in tori.values():
        t.close()
    assert not failures, f"{len(failures)} mismatches, first: {failures[:5]}"


@pytest.mark.parametrize("engine", ENGINES)
def test_anchors(ltl, orc, engine):
    for a in load("anchors.json")["anchors"]:
        init = orc.init_random(a["n"], a["density"], a["seed"])
        out = ltl.run_engine(engine, init, a["rule"], a["steps"])
        assert int(out.sum()) == a["alive"], a
        assert _fnv(orc, out) == a["fnv"], a


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("rows,cols", [(96, 160), (200, 72), (33, 1000), (4096, 128), (17, 17)])
def test_rectangular_torus(ltl, orc, engine, rows, cols):
    rng = np.random.default_rng(rows * 7 + cols)
    init = (rng.random((rows, cols)) < 0.3).astype(np.uint8)
    for text in ("R1,C2,M0,S2..3,B3..3,NM", "R7,C2,M1,S60..140,B50..110,NM",
                 "R16,C2,M0,S170..296,B170..300,NM", "R9,C2,M0,S5..18,B7..12,NN"):
        rule = parse_rule_text(text)
        with ltl.DeviceTorus(rows=rows, cols=cols) as t:
            t.upload(init)
            t.run(text, 3, engine=engine)
            got = t.download()
        assert np.array_equal(got, orc.simulate(init, rule, 3)), (text, rows, cols)


def test_max_h_max_r_all_alive(ltl):
    """acceptance.cpp:245-277: all-live grid at r=16 hits H=33 and R=1089 exactly."""
    for engine in ENGINES:
        g = np.ones((64, 64), np.uint8)
        _, st = ltl.run_engine(engine, g, "R16,C2,M1,S0..1089,B0..1089,NM", 1, stats=True)
        assert (st["max_h"], st["max_r"]) == (33, 1089), engine


def test_mma_accounting_matches_reference(ltl, orc):
    """CatStats.mma_count in reference fragment units (test_cat_engine.cpp:274-305)."""
    for c in load("criterion1.json")["cases"][:40]:
        init = orc.init_random(c["n"], c["density"], c["seed"])
        _, st = ltl.run_engine("cat", init, c["rule"], c["steps"], f=c["f"], stats=True)
        assert st["mma_count"] == c["mma_count"]
        assert st["max_h"] == c["max_h"] and st["max_r"] == c["max_r"], c


def test_fault_injection_detected(ltl, orc):
    """test_cat_engine.cpp:353-370: a corrupted band entry must diverge or trip the guard."""
    init = orc.init_random(64, 0.3, 1)
    rule = "R1,C2,M0,S2..3,B3..3,NM"
    clean = ltl.run_engine("cat", init, rule, 5)
    try:
        faulty = ltl.run_engine("cat", init, rule, 5, inject_fault=True)
        assert not np.array_equal(faulty, clean)
    except ltl.LtlLogicError as e:
        assert "internal consistency: negative neighborhood count" in str(e)


def test_fault_injection_matches_reference(ltl, orc):
    """CatConfig.inject_band_fault flips pi2(0,0) of every band fragment
    (src/cat_engine.cpp:277): the faulted tcgen05 run must reproduce the
    reference's faulted run byte for byte -- the same diverged grid, or the
    same negative-count abort (tests/golden/faults.json, made by the reference)."""
    bad = []
    for c in load("faults.json")["cases"]:
        init = orc.init_random(c["n"], c["density"], c["seed"])
        with ltl.DeviceTorus(n=c["n"], f=c["f"]) as t:
            t.upload(init)
            try:
                t.run(c["rule"], c["steps"], inject_fault=True)
                got = dict(alive=int(t.download().sum()), fnv=_fnv(orc, t.download()))
            except ltl.LtlLogicError as e:
                got = dict(error=str(e))
        want = {k: c[k] for k in ("alive", "fnv", "error") if k in c}
        if got != want:
            bad.append((c["rule"], c["n"], c["f"], c["steps"], want, got))
    assert not bad, f"{len(bad)} mismatches, first: {bad[:3]}"


def test_virtual_slabs_match_single(ltl, orc):
    """The multi-GPU slab path (halo rows exchanged between slabs) with every slab
    on device 0: bit-identical to one slab and to the oracle."""
    init = orc.init_random(512, 0.26, 3)
    text = "R16,C2,M0,S170..296,B170..300,NM"
    expect = orc.simulate(init, parse_rule_text(text), 6)
    for slabs in (1, 2, 3, 4, 8):
        with ltl.DeviceTorus(n=512, slabs=slabs, devices=[0] * slabs) as t:
            t.upload(init)
            t.run(text, 6)
            assert np.array_equal(t.download(), expect), slabs


def test_steps_zero_is_identity(ltl, orc):
    init = orc.init_random(64, 0.5, 2)
    assert np.array_equal(ltl.run_engine("cat", init, "R2,C2,M0,S7..12,B8..11,NM", 0), init)


def test_run_errors(ltl):
    with ltl.DeviceTorus(n=32, f=4) as t:
        with pytest.raises(ValueError, match="unsupported radius r=5 for fragment side f=4"):
            t.run("R5,C2,M0,S35..59,B34..45,NM", 1)
        with pytest.raises(ValueError, match="config error: steps must be >= 0"):
            t.run("R1,C2,M0,S2..3,B3..3,NM", -1)


def test_large_grid_engines_agree(ltl, orc):
    """At sizes the oracle is slow for: tcgen05 == base == pack == oracle on a
    4096^2 grid for a few generations, at three radii."""
    init = orc.init_random(4096, 0.3, 11)
    for text in ("R1,C2,M0,S2..3,B3..3,NM", "R5,C2,M1,S34..58,B34..45,NM",
                 "R16,C2,M0,S170..296,B170..300,NM"):
        a = ltl.run_engine("cat", init, text, 2)
        for engine in ("base", "pack"):
            assert np.array_equal(a, ltl.run_engine(engine, init, text, 2)), (engine, text)
        assert np.array_equal(a, orc.simulate(init, parse_rule_text(text), 2)), text


def test_device_init_random_matches_reference(ltl, orc):
    """Device init_random == the reference's splitmix64 grid (src/grid.cpp:61-73),
    including fill_n padding and density edges."""
    from golden_data import unpack_grid
    for e in load("kats.json")["init_grids"]:
        with ltl.DeviceTorus(n=e["n"], f=e["f"]) as t:
            t.init_random(e["density"], e["seed"], e["fill_n"])
            assert np.array_equal(t.download(), unpack_grid(e)), e
    for n, d, seed in ((1024, 0.5, 1), (333, 0.37, 99), (64, 0.0, 5), (64, 1.0, 5),
                       (128, 2.0 ** -70, 0)):
        with ltl.DeviceTorus(rows=n, cols=n) as t:
            t.init_random(d, seed)
            assert np.array_equal(t.download(), orc.init_random(n, d, seed)), (n, d, seed)


def test_partition_single_rank_matches_torus(ltl, orc):
    """The multi-process slab path (ltl_create_part + ltl_step_part + the row
    exchange of paper_2406_17284_b200.dist) at world size 1."""
    from paper_2406_17284_b200.dist import PartitionedTorus
    part = PartitionedTorus(256, 192, 0, 1, 0)
    part.init_random(0.21, 1)
    text = "R5,C2,M1,S34..58,B34..45,NM"
    for _ in range(5):
        part.step(text)
    part.torus.synchronize()
    init = np.zeros((256, 192), np.uint8)
    with ltl.DeviceTorus(rows=256, cols=192) as t:
        t.init_random(0.21, 1)
        init = t.download()
    assert np.array_equal(part.torus.download(), orc.simulate(init, parse_rule_text(text), 5))


@pytest.mark.parametrize("rows,cols", [(128, 128), (96, 256), (160, 384), (224, 128),
                                       (200, 256), (128, 200), (64, 1024)])
def test_wrap_by_load_geometries(ltl, orc, rows, cols):
    """The step's own periodic wrap (side boxes of strip 0 / S-1 taken from the
    other end, first / last band boxes assembled from two pieces) against the
    oracle, on aligned and unaligned tori (these fall back to the halo kernel
    for the unaligned direction), several generations, Moore and VN."""
    rng = np.random.default_rng(rows * 31 + cols)
    init = (rng.random((rows, cols)) < 0.3).astype(np.uint8)
    for text in ("R1,C2,M0,S2..3,B3..3,NM", "R16,C2,M0,S170..296,B170..300,NM",
                 "R9,C2,M0,S5..18,B7..12,NN"):
        with ltl.DeviceTorus(rows=rows, cols=cols) as t:
            t.upload(init)
            t.run(text, 5)
            got = t.download()
        assert np.array_equal(got, orc.simulate(init, parse_rule_text(text), 5)), (text, rows, cols)


@pytest.mark.parametrize("rows,cols", [(128, 128), (256, 256), (1024, 1024), (512, 384)])
def test_persistent_multi_generation(ltl, orc, rows, cols, monkeypatch):
    """Multi-generation launches (units handed between generations through
    per-unit flags) forced on small tori: odd and even generation counts equal
    the oracle, Moore and VN, and a second run on the same context continues
    from the flags' new base."""
    monkeypatch.setenv("LTL_FORCE_PERSIST", "1")
    rng = np.random.default_rng(rows + 3 * cols)
    init = (rng.random((rows, cols)) < 0.3).astype(np.uint8)
    for text in ("R5,C2,M1,S34..58,B34..45,NM", "R7,C2,M0,S5..15,B4..10,NN"):
        rule = parse_rule_text(text)
        with ltl.DeviceTorus(rows=rows, cols=cols) as t:
            t.upload(init)
            t.run(text, 7)
            assert np.array_equal(t.download(), orc.simulate(init, rule, 7)), (text, 7)
            t.run(text, 6)
            assert np.array_equal(t.download(), orc.simulate(init, rule, 13)), (text, 13)


def test_persistent_full_gpu_equals_per_generation(ltl, monkeypatch):
    """n = 148 x 128 (units per SM in the sweep range), so ltl_run takes the
    multi-generation launch by default; bit-identical to one launch per
    generation (LTL_NO_PERSIST)."""
    import torch
    n = 128 * torch.cuda.get_device_properties(0).multi_processor_count
    text = "R5,C2,M1,S34..58,B34..45,NM"
    outs = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("LTL_NO_PERSIST", env)
        with ltl.DeviceTorus(rows=n, cols=n) as t:
            t.init_random(0.21, 1)
            t.run(text, 5)
            outs.append(t.download())
    assert np.array_equal(outs[0], outs[1])


def test_stencil_after_tcgen05_refreshes_halo(ltl, orc):
    """tcgen05 generations leave the halo cells they do not need stale; a
    stencil generation on the same context must refresh them first."""
    init = orc.init_random(256, 0.3, 4)
    text = "R4,C2,M0,S10..20,B8..12,NM"
    with ltl.DeviceTorus(n=256) as t:
        t.upload(init)
        t.run(text, 3)
        t.run(text, 2, engine="base")
        t.run(text, 1)
        t.run(text, 1, engine="pack")
        got = t.download()
    assert np.array_equal(got, orc.simulate(init, parse_rule_text(text), 7))


def test_partition_wrap_cols_matches_torus(ltl, orc):
    """The multi-process slab path on a 128-aligned width (column wrap by the
    step's loads, rows by pack/exchange/unpack) at world size 1."""
    from paper_2406_17284_b200.dist import PartitionedTorus
    part = PartitionedTorus(384, 256, 0, 1, 0)
    part.init_random(0.3, 2)
    text = "R16,C2,M0,S170..296,B170..300,NM"
    for _ in range(4):
        part.step(text)
    part.torus.synchronize()
    with ltl.DeviceTorus(rows=384, cols=256) as t:
        t.init_random(0.3, 2)
        init = t.download()
    assert np.array_equal(part.torus.download(), orc.simulate(init, parse_rule_text(text), 4))


@pytest.mark.parametrize("rows,cols", [(256, 256), (512, 384)])
def test_persistent_self_ring(ltl, orc, rows, cols, monkeypatch):
    """Multi-generation launches of a ring slab (here its own neighbour): the
    first / last band wait on the neighbours' unit counters (system scope) and
    read their rows out of the neighbour's buffers; two calls in a row."""
    monkeypatch.setenv("LTL_SELF_RING", "1")
    monkeypatch.setenv("LTL_FORCE_PERSIST", "1")
    rng = np.random.default_rng(rows + cols)
    init = (rng.random((rows, cols)) < 0.3).astype(np.uint8)
    for text in ("R5,C2,M1,S34..58,B34..45,NM", "R7,C2,M0,S5..15,B4..10,NN"):
        rule = parse_rule_text(text)
        with ltl.DeviceTorus(rows=rows, cols=cols) as t:
            assert t.ring_active()
            t.upload(init)
            t.run(text, 7)
            assert np.array_equal(t.download(), orc.simulate(init, rule, 7)), (text, 7)
            t.run(text, 6)
            assert np.array_equal(t.download(), orc.simulate(init, rule, 13)), (text, 13)


def test_persistent_sweep_all_radii(ltl, orc, monkeypatch):
    """The multi-generation sweep (forced onto a 384 x 256 torus: 3 bands x 2
    strips) for every preset radius 1..16 and von Neumann probes, against the
    oracle."""
    monkeypatch.setenv("LTL_FORCE_PERSIST", "1")
    rng = np.random.default_rng(5)
    cases = [(text, dens) for _, text, dens in ltl.ltl_presets()]
    cases += [(ltl.format_ltl_rule(ltl.von_neumann_probe_rule(r)), 0.25) for r in (1, 8, 16)]
    for text, dens in cases:
        init = (rng.random((384, 256)) < dens).astype(np.uint8)
        with ltl.DeviceTorus(rows=384, cols=256) as t:
            t.upload(init)
            t.run(text, 6)
            got = t.download()
        assert np.array_equal(got, orc.simulate(init, parse_rule_text(text), 6)), text


def test_bench_geometry_persistent_vs_stencil(ltl, orc):
    """The bench workload itself (configs[1]: Bosco r=5 on 16384^2, the
    persistent sweep by default) against the CUDA-core stencil engine, which
    is pinned to the oracle above: 4 generations."""
    n, text = 16384, "R5,C2,M1,S34..58,B34..45,NM"
    with ltl.DeviceTorus(n=n) as t:
        t.init_random(0.21, 1)
        init = t.download()
        t.run(text, 4)
        tc = t.download()
    with ltl.DeviceTorus(n=n) as t:
        t.upload(init)
        t.run(text, 4, engine="pack")
        st = t.download()
    assert np.array_equal(tc, st)
    assert 0 < int(tc.sum()) < n * n


@pytest.mark.parametrize("kind", ["R16,C2,M0,S170..296,B170..300,NM", "R11,C2,M0,S5..21,B9..16,NN"])
def test_determinism_matrix(ltl, orc, kind, monkeypatch):
    """acceptance.cpp:352-384 analogue for the device schedule: the CTA count
    (LTL_TC_GRID in {1, 7, 64, 148}) and the multi-generation sweep's chunk
    length (LTL_SWEEP_UNITS in {1, 5, 12}) must not change a single byte --
    per-launch and persistent paths, against one oracle-checked run."""
    n, steps = 1024, 5
    init = orc.init_random(n, 0.3, 9)
    expect = orc.simulate(init, parse_rule_text(kind), steps)
    for persist in ("0", "1"):
        monkeypatch.setenv("LTL_FORCE_PERSIST" if persist == "1" else "LTL_NO_PERSIST", "1")
        monkeypatch.delenv("LTL_NO_PERSIST" if persist == "1" else "LTL_FORCE_PERSIST",
                           raising=False)
        for grid in ("1", "7", "64", "148"):
            for units in ("1", "5", "12"):
                monkeypatch.setenv("LTL_TC_GRID", grid)
                monkeypatch.setenv("LTL_SWEEP_UNITS", units)
                with ltl.DeviceTorus(rows=n, cols=n) as t:
                    t.upload(init)
                    t.run(kind, steps)
                    got = t.download()
                assert np.array_equal(got, expect), (kind, persist, grid, units)
                if persist == "0":
                    break  # the chunk length only matters to the sweep


@pytest.mark.parametrize("grid", ["3", "5", "7"])
def test_dynamic_schedule_matches_static(ltl, orc, grid, monkeypatch):
    """One launch per generation with whole-band rounds hands the remainder out
    at run time (ltl_tc.cu SegIter<kDyn>); CTA counts that leave a remainder of
    1..3 bands: the same bytes, H / R maxima and faulted grids as the static
    schedule and the oracle."""
    n, text = 1024, "R7,C2,M1,S60..140,B50..110,NM"
    init = orc.init_random(n, 0.3, 4)
    monkeypatch.setenv("LTL_NO_PERSIST", "1")
    monkeypatch.setenv("LTL_TC_GRID", grid)
    outs = []
    for static in (False, True):
        if static:
            monkeypatch.setenv("LTL_STATIC_SCHED", "1")
        with ltl.DeviceTorus(n=n) as t:
            t.upload(init)
            st = t.run(text, 3, stats=True)
            got = t.download()
            t.upload(init)
            try:
                t.run(text, 2, inject_fault=True)
                faulted = t.download()
            except ltl.LtlLogicError as e:
                faulted = str(e)
        outs.append((got, st["max_h"], st["max_r"], faulted))
    assert np.array_equal(outs[0][0], orc.simulate(init, parse_rule_text(text), 3))
    assert np.array_equal(outs[0][0], outs[1][0]) and outs[0][1:3] == outs[1][1:3]
    f0, f1 = outs[0][3], outs[1][3]
    assert (isinstance(f0, str) and f0 == f1) or np.array_equal(f0, f1)
