"""In-tree build of libltl_b200.so (sm_100a) -- no JIT cache, no site-packages.

    python -m paper_2406_17284_b200._build         # or __graft_entry__.build()

Every .cu under csrc/ is compiled by nvcc for ``-gencode
arch=compute_100a,code=sm_100a`` with ``-lineinfo`` (so ncu's source page maps
to our lines) and linked with the static CUDA runtime, so the library has no
link-time dependency on libcuda/libcudart and loads on GPU-less hosts.  The
ptxas resource report (registers, spills, smem) lands in build/ptxas.log.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "ltl_b200")
LIB = os.path.join(PKG, "libltl_b200.so")
CLI_SRC = os.path.join(PKG, "cli", "catbench.cpp")
CLI = os.path.join(PKG, "bin", "catbench")  # the reference's CLI over include/catsim

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-Wall",
          "-I", os.path.join(ROOT, "include"), "-I", CSRC]
# extra nvcc flags for diagnostics builds, e.g. LTL_NVCC_FLAGS=-DLTL_TC_TRACE_BUILD
COMMON += os.environ.get("LTL_NVCC_FLAGS", "").split()


def sources():
    cu = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    cpp = sorted(glob.glob(os.path.join(CSRC, "host", "*.cpp")))
    return cu, cpp


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _headers():
    return (glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "host", "*.hpp"))
            + glob.glob(os.path.join(ROOT, "include", "*.h"))
            + glob.glob(os.path.join(ROOT, "include", "catsim", "*.hpp")))


def _compile(src: str, obj: str) -> str:
    if src.endswith(".cu"):
        cmd = [NVCC, *ARCH, *COMMON, "-Xptxas", "-v", "-c", src, "-o", obj]
    else:
        cmd = [NVCC, *ARCH, *COMMON, "-x", "c++", "-c", src, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    return res.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    # objects built with other extra flags (LTL_NVCC_FLAGS) are stale too
    stamp = os.path.join(BUILD, "flags.txt")
    flags = " ".join(COMMON)
    try:
        with open(stamp) as fh:
            force = force or fh.read() != flags
    except OSError:
        force = True
    with open(stamp, "w") as fh:
        fh.write(flags)
    cu, cpp = sources()
    hdrs = _headers()
    jobs, objs = [], []
    for src in cu + cpp:
        rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
        obj = os.path.join(BUILD, rel + ".o")
        objs.append(obj)
        if force or _newer(obj, [src, *hdrs]):
            jobs.append((src, obj))
    logs = []
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            for src, log in zip([j[0] for j in jobs], ex.map(lambda j: _compile(*j), jobs)):
                logs.append(f"== {os.path.relpath(src, ROOT)}\n{log}")
        with open(os.path.join(ROOT, "build", "ptxas.log"), "w") as fh:
            fh.write("\n".join(logs))
    if force or jobs or _newer(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs,
               "-Xlinker", "--no-undefined", "-ldl", "-lpthread", "-lrt"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    if force or _newer(CLI, [CLI_SRC, LIB, *hdrs]):
        os.makedirs(os.path.dirname(CLI), exist_ok=True)
        cxx = shutil.which("g++") or "g++"
        cmd = [cxx, "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
               CLI_SRC, "-o", CLI, f"-L{PKG}", "-lltl_b200", "-Wl,-rpath,$ORIGIN/.."]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"catbench build failed: {' '.join(cmd)}\n{res.stderr}")
    if verbose:
        print("\n".join(logs))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
