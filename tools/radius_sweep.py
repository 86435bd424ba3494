"""Config 3 of BASELINE.json: radius sweep r = 1..16 on one B200.

For every radius the published preset of that radius (Table III,
proj/src/rule.cpp:113-133) at its seeding density, on an n x n torus
(default 32768, configs[2]):
  * tcgen05 banded-MMA step    (device-timed, CUDA events)
  * CUDA-core stencil ablation (device-timed)
  * the reference's CPU CAT engine on this host's cores (oracle/_ref; a bounded
    sample: `--cpu-n` square grid, 2 generations; the CPU rate is flat in n)
plus a bit-exactness spot check of tcgen05 == stencil on the full grid.

    python tools/radius_sweep.py [--n 32768] [--steps 50] [--out profiles/radius_sweep_r01.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--stencil-steps", type=int, default=3)
    ap.add_argument("--cpu-n", type=int, default=2048)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--radii", default="1-16")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "radius_sweep_r01.json"))
    args = ap.parse_args()
    from paper_2406_17284_b200 import ltl

    lo, hi = (int(v) for v in args.radii.split("-"))
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
        hbm = json.load(fh)["hbm_gbs"]
    ref = None
    if not args.no_cpu:
        import oracle
        ref = oracle.Reference()
    presets = ltl.ltl_presets()
    n = args.n
    cells = n * n
    torus = ltl.DeviceTorus(rows=n, cols=n)
    rows = []
    for r in range(lo, hi + 1):
        name, rule, dens = presets[r - 1]
        torus.init_random(dens, 1)
        tc_total, tc_kernel = torus.time(rule, args.steps, 3)
        a = torus.download()
        torus.init_random(dens, 1)
        st_total, st_kernel = torus.time(rule, args.stencil_steps, 1, stencil=True)
        # parity spot check on the full grid: same start, 2 generations each engine
        torus.init_random(dens, 1)
        torus.run(rule, 2)
        g_tc = torus.download()
        torus.init_random(dens, 1)
        torus.run(rule, 2, stencil=True)
        g_st = torus.download()
        row = {
            "r": r, "preset": name, "rule": rule, "density": dens, "n": n,
            "tc_cells_per_s": cells * args.steps / (tc_total / 1e3),
            "tc_kernel_us": tc_kernel * 1e3 / args.steps,
            "tc_hbm_frac": 2 * cells / (tc_kernel / 1e3 / args.steps) / 1e9 / hbm,
            "stencil_cells_per_s": cells * args.stencil_steps / (st_total / 1e3),
            "stencil_kernel_us": st_kernel * 1e3 / args.stencil_steps,
            "tc_equals_stencil_2gen": bool(np.array_equal(g_tc, g_st)),
        }
        row["tc_over_stencil"] = row["tc_cells_per_s"] / row["stencil_cells_per_s"]
        if ref is not None:
            cg = ref.init_random(args.cpu_n, dens, 1)
            cores = max(1, ref.hardware_concurrency())
            t0 = time.perf_counter()
            ref.run_engine("cat", cg, rule, 2, workers=cores)
            row["cpu_cells_per_s"] = args.cpu_n ** 2 * 2 / (time.perf_counter() - t0)
            row["cpu_cores"] = cores
            row["tc_over_cpu"] = row["tc_cells_per_s"] / row["cpu_cells_per_s"]
        rows.append(row)
        print(json.dumps(row), flush=True)
    out = {"config": f"BASELINE configs[2]: radius sweep, {n}x{n}, presets r={lo}..{hi}",
           "hbm_peak_gbs": hbm, "tc_steps": args.steps, "stencil_steps": args.stencil_steps,
           "cpu_sample": f"{args.cpu_n}^2 grid, 2 generations of run_engine(Cat), all host cores",
           "rows": rows}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)
    tcs = [x["tc_cells_per_s"] for x in rows]
    print(f"tc cells/s min {min(tcs):.3e} max {max(tcs):.3e} spread {(max(tcs) / min(tcs) - 1) * 100:.1f}%")


if __name__ == "__main__":
    main()
