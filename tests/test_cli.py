"""catbench (paper_2406_17284_b200/cli/catbench.cpp): the reference's CLI
(proj/tools/catbench.cpp) over include/catsim and the B200 engines.

The reference's nine CLI smoke tests (proj/tests/CMakeLists.txt:23-46) are
reproduced verbatim as command lines with their expected exit status
(`cli_bad_engine` must FAIL: `--engine gpu` is not an engine); argument errors
run on the CPU, everything that touches a grid on the GPU."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2406_17284_b200", "bin", "catbench")

# proj/tests/CMakeLists.txt:23-46: (name, argv, must_fail)
REFERENCE_SMOKE = [
    ("cli_run_smoke", ["run", "--preset", "life", "--n", "64", "--steps", "4"], False),
    ("cli_run_rounding", ["run", "--rule", "R2,C2,M0,S7..12,B8..11,NM", "--n", "50",
                          "--steps", "2", "--engine", "base"], False),
    ("cli_verify_smoke", ["verify", "--radii", "1,2", "--sizes", "32", "--seeds", "1"], False),
    ("cli_verify_fault", ["verify", "--radii", "1", "--sizes", "32", "--seeds", "1", "--kinds",
                          "vn", "--steps", "2", "--inject-fault"], False),
    ("cli_bench_smoke", ["bench", "--preset", "life", "--n", "128", "--steps", "2",
                         "--max-realizations", "3", "--target-stderr", "100"], False),
    ("cli_sweep_smoke", ["sweep-tiles", "--preset", "life", "--n", "128", "--steps", "2",
                         "--realizations", "1", "--shapes", "1x14,4x4"], False),
    ("cli_cost_model", ["cost-model"], False),
    ("cli_cost_model_derive", ["cost-model", "--set", "w=16", "--set", "h=16", "--derive-e",
                               "16", "14.8"], False),
    ("cli_bad_engine", ["run", "--preset", "life", "--engine", "gpu"], True),
]


def run(args, timeout=600, env=None):
    if not os.path.exists(CLI):
        pytest.skip("catbench not built (python -m paper_2406_17284_b200._build)")
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=timeout, env=env)


def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


# ---- argument handling (no device needed) ---------------------------------
def test_bad_engine_fails_before_any_device_work():
    res = run(["run", "--preset", "life", "--engine", "gpu"])
    assert res.returncode == 2
    assert "config error: unknown engine 'gpu' (cat, base, pack)" in res.stderr


@pytest.mark.parametrize("args,code", [
    ([], 106),                                   # a subcommand is required
    (["frobnicate"], 109),                       # unknown subcommand
    (["run", "--bogus", "1"], 109),              # unknown option
    (["run", "--f", "5"], 105),                  # --f not in {4,8,16}
    (["run", "--n", "abc"], 104),                # not a number
    (["run", "--n"], 114),                       # missing value
    (["run", "--rule", "R1,C2,M0,S2..3,B3..3,NM", "--preset", "life"], 2),
    (["run", "--preset", "nope"], 2),
    (["run", "--rule", "R0,C2,M0,S2..3,B3..3,NM"], 2),
    (["verify", "--radii", "17"], 2),
    (["verify", "--radii", "3-1"], 2),
    (["sweep-tiles", "--shapes", "4"], 2),
])
def test_argument_errors(args, code):
    res = run(args)
    assert res.returncode == code, (res.stdout, res.stderr)


def test_help():
    res = run(["--help"])
    assert res.returncode == 0 and "usage: catbench" in res.stdout


def test_error_messages_are_the_references():
    assert "config error: --rule and --preset are mutually exclusive" in run(
        ["run", "--rule", "R1,C2,M0,S2..3,B3..3,NM", "--preset", "life"]).stderr
    assert "config error: unknown preset 'nope' (known: life, " in run(
        ["run", "--preset", "nope"]).stderr
    assert "unsupported rule: radius 0 outside 1..16" in run(
        ["run", "--rule", "R0,C2,M0,S2..3,B3..3,NM"]).stderr


# ---- the reference's CLI smoke tests, on the GPU ---------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("name,args,must_fail", REFERENCE_SMOKE, ids=[t[0] for t in REFERENCE_SMOKE])
def test_reference_cli_smoke(name, args, must_fail):
    _gpu()
    res = run(args)
    if must_fail:
        assert res.returncode != 0, res.stdout
    else:
        assert res.returncode == 0, (res.stdout, res.stderr)


@pytest.mark.gpu
def test_run_matches_reference(tmp_path, ref):
    """`catbench run` output lines and its --out snapshot against the unmodified
    reference's run_engine + snapshot_write on the same seed / rule."""
    _gpu()
    snap = tmp_path / "final.bin"
    res = run(["run", "--preset", "bosco", "--n", "200", "--steps", "9", "--seed", "3",
               "--out", str(snap)])
    assert res.returncode == 0, res.stderr
    lines = res.stdout.splitlines()
    assert lines[0] == ("engine cat rule R5,C2,M0,S35..59,B34..45,NM n 208 (requested 200, "
                        "padded to fit f) f 16 steps 9 seed 3 density 0.21")
    init = ref.init_random(208, 0.21, 3, 16, 200)
    want = ref.run_engine("cat", init, "R5,C2,M0,S35..59,B34..45,NM", 9)
    assert lines[1] == f"alive {int(want.sum())}"
    assert re.match(r"elapsed_ms [0-9.]+ ms_per_step [0-9.]+ cells_per_sec [0-9.e+]+$", lines[2])
    _, st = ref.run_engine("cat", init, "R5,C2,M0,S35..59,B34..45,NM", 9, stats=True)
    assert lines[3] == f"mma_count {st['mma_count']} max_h {st['max_h']} max_r {st['max_r']}"
    assert lines[4] == f"snapshot {snap}"
    ref_snap = tmp_path / "ref.bin"
    ref.snapshot_write(want, str(ref_snap))
    assert snap.read_bytes() == ref_snap.read_bytes()


@pytest.mark.gpu
def test_run_base_reports_memory_accesses(ref):
    _gpu()
    res = run(["run", "--rule", "R2,C2,M0,S7..12,B8..11,NM", "--n", "50", "--steps", "2",
               "--engine", "base"])
    assert res.returncode == 0, res.stderr
    init = ref.init_random(64, 0.25, 1, 16, 50)
    _, st = ref.run_engine("base", init, "R2,C2,M0,S7..12,B8..11,NM", 2, stats=True)
    assert f"memory_accesses {st['accesses']}" in res.stdout
    want = ref.run_engine("base", init, "R2,C2,M0,S7..12,B8..11,NM", 2)
    assert f"alive {int(want.sum())}" in res.stdout


@pytest.mark.gpu
def test_verify_output():
    _gpu()
    res = run(["verify", "--radii", "1,9,16", "--sizes", "32,64", "--seeds", "1,2"])
    assert res.returncode == 0, res.stdout[-3000:]
    lines = res.stdout.splitlines()
    assert lines[-1] == "verified 48 combinations: 48 pass, 0 fail"
    assert "PASS r=1 kind=moore n=32 seed=1 steps=1 engines=cat,base,pack" in lines
    assert all(l.startswith("PASS ") for l in lines[:-1])
    # the faulted band (pi2(0,0) flipped) escapes detection in exactly the
    # two combinations where it also escapes in the reference (oracle/_ref,
    # run_engine(Cat, inject_band_fault) vs run_engine(Base), same seeds)
    res = run(["verify", "--radii", "1-4", "--sizes", "32", "--seeds", "1", "--inject-fault"])
    assert res.returncode == 1
    assert res.stdout.splitlines()[-1] == "verified 16 combinations: 14 pass, 2 fail"
    assert [l for l in res.stdout.splitlines() if l.startswith("FAIL")] == [
        "FAIL r=2 kind=moore n=32 seed=1 steps=25 (fault missed)",
        "FAIL r=4 kind=moore n=32 seed=1 steps=25 (fault missed)"]


@pytest.mark.gpu
def test_bench_csv(tmp_path):
    _gpu()
    out = tmp_path / "b.csv"
    res = run(["bench", "--preset", "globe", "--n", "256", "--steps", "3", "--max-realizations",
               "3", "--target-stderr", "100", "--csv", str(out)])
    assert res.returncode == 0, res.stderr
    assert res.stdout.strip() == f"wrote {out}"
    rows = out.read_text().splitlines()
    assert rows[0] == "engine,n,r,steps,realizations,ms_per_step,stderr_pct,cells_per_sec"
    assert [r.split(",")[0] for r in rows[1:]] == ["cat", "base", "pack"]
    for r in rows[1:]:
        f = r.split(",")
        assert f[1:5] == ["256", "8", "3", "3"]
        assert np.isclose(float(f[7]), 256 * 256 * 1000.0 / float(f[5]), rtol=1e-4)


# ---- cost-model (pure host: runs on the CPU) -------------------------------
def test_cost_model_table_cpu():
    """catbench cost-model: the paper's Table II from the restated model."""
    res = run(["cost-model", "--csv"])
    assert res.returncode == 0, res.stderr
    rows = [r.split(",") for r in res.stdout.strip().splitlines()]
    assert rows[0] == ["scenario", "r=1", "r=4", "r=8", "r=16"]
    published = {"GH100 Chip": [1.20, 8.07, 27.9, 104.0], "More TC Units": [1.59, 10.6, 37.1, 138.0],
                 "Faster TC Units": [1.55, 10.4, 36.1, 134.0], "More FP Units": [0.60, 4.06, 14.1, 52.5],
                 "Regular Tiles": [0.17, 1.15, 3.99, 14.8], "Expensive f()": [0.79, 1.17, 2.25, 6.44]}
    assert [r[0] for r in rows[1:]] == list(published)
    for r in rows[1:]:
        for got, want in zip(map(float, r[1:]), published[r[0]]):
            assert abs(got - want) <= 0.02 * want, (r[0], got, want)
    text = run(["cost-model"]).stdout
    assert "speedup limit vs per-cell reference" in text and "GH100 Chip" in text


def test_cost_model_derive_cpu():
    res = run(["cost-model", "--set", "w=16", "--set", "h=16", "--derive-e", "16", "14.8"])
    assert res.returncode == 0, res.stderr
    assert res.stdout.startswith("E=9.33700")
    res = run(["cost-model", "--derive-e", "1", "100"])
    assert res.returncode == 2 and "infeasible" in res.stderr
    res = run(["cost-model", "--set", "bogus=1"])
    assert res.returncode == 2 and "unknown parameter" in res.stderr
