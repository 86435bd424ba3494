"""The catsim C++ API (include/catsim/, header-only over the C-ABI) compiled the
way a reference user would compile it, running the reference's own engine /
grid / snapshot test cases (tests/cpp/test_catsim_api.cpp) plus the
reference-generated anchors of tests/golden/anchors.json."""
import json
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_catsim_api.cpp")
LIBDIR = os.path.join(ROOT, "paper_2406_17284_b200")
CXX = shutil.which("g++") or os.environ.get("CXX", "g++")


def compile_test(out):
    from paper_2406_17284_b200 import ltl
    ltl.load_library()  # the in-tree .so must exist
    cmd = [CXX, "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", f"-I{ROOT}/include", SRC,
           f"-L{LIBDIR}", "-lltl_b200", f"-Wl,-rpath,{LIBDIR}", "-o", str(out)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr[-4000:]


def test_cpp_api_compiles_and_links(tmp_path):
    compile_test(tmp_path / "test_catsim_api")


@pytest.mark.gpu
def test_cpp_api_reference_cases(tmp_path):
    exe = tmp_path / "test_catsim_api"
    compile_test(exe)
    with open(os.path.join(ROOT, "tests", "golden", "anchors.json")) as fh:
        anchors = json.load(fh)["anchors"]
    args = []
    for a in anchors:
        if "cat" not in a.get("engines", ["cat"]):
            continue
        args += [a["rule"], str(a["n"]), repr(a["density"]), str(a["seed"]), str(a["steps"]),
                 str(a["alive"]), a["fnv"]]
    res = subprocess.run([str(exe), os.path.join(ROOT, "tests", "golden", "snapshots"),
                          str(tmp_path), *args], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, (res.stdout + res.stderr)[-4000:]
    assert "0 failed" in res.stdout
