"""bench.py's contract where it runs without a GPU: the reference arm (the
reference's own CPU CAT engine, oracle/_ref) prints one JSON line with the
keys the driver reads, on the same metric / unit / config as the GPU arm."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ref_line(*args):
    import oracle
    if not os.path.exists(oracle.REF_SO):
        pytest.skip("oracle/_ref not built")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          *args], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _ref_line("--workload", "c0", "--steps", "2", "--warmup", "3")
    assert d["impl"] == "reference"
    assert d["metric"] == "cell updates/sec vs radius r=1..16 at 1/2/4/8 B200; % of roofline"
    assert d["unit"] == "cell updates/s" and d["higher_is_better"] is True
    assert d["steps"] == 2 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["value"] == d["value"] and cb["cores"] >= 1
    assert d["config"]["workload"].startswith("configs[0]") and d["config"]["n"] == 1024


def test_reference_arm_multi_gpu_line_is_rank0_only():
    """--gpus N without torchrun: the reference arm is CPU work on rank 0 only,
    on the N-GPU workload (configs[4], a bounded 16384^2 sample of its rule)."""
    d = _ref_line("--gpus", "2", "--steps", "1", "--warmup", "3")
    assert d["n_gpus"] == 2 and d["config"]["workload"].startswith("configs[4]")
    assert "bounded sample" in d["cpu_baseline"]["sample"]
