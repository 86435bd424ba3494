#!/usr/bin/env python
"""bench.py -- cell updates/s of the B200 LTL step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): Bosco's rule as BASELINE states it,
R5,C2,M1,S34..58,B34..45,NM, on a 16384 x 16384 torus seeded by init_random
(density 0.21, seed 1; generated on the device, bit-identical to the
reference's splitmix64 grid).  One bench step = one generation of the whole
torus (configs[1] runs 1000 of them, the default K).  With N GPUs
(torchrun, one process per GPU) every rank owns a 16384 x 16384 row slab of an
(N*16384) x 16384 torus and exchanges 16 halo rows per generation with its
ring neighbours over NCCL: weak scaling.

Rank 0 prints ONE JSON line.  `value` is device-timed (CUDA events on the
launching stream, max over ranks) with the grid resident in HBM; the two
256 MiB generation buffers exceed the 126 MB L2, so no flush is needed.
`e2e` is the same metric through the public C-ABI call a user makes
(ltl_run_interior = run_engine(Cat): upload from pinned host memory, K
generations, download), wall-clocked.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

RULE = "R5,C2,M1,S34..58,B34..45,NM"
N_SIDE = 16384
DENSITY = 0.21
SEED = 1
METRIC = "cell updates/sec vs radius r=1..16 at 1/2/4/8 B200; % of roofline"
UNIT = "cell updates/s"
BYTES_PER_CELL = 2  # read 1 B state + write 1 B next state


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def ncu_traffic():
    """dram read+write bytes per generation of the step kernel from the
    committed ncu --set full capture (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_tc_step.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get("dram_bytes_per_generation"), d.get("n")
    except (OSError, ValueError):
        return None, None


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons, watts = [], 0, set(), []
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        with open(self.path) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx = max(mx, float(parts[2]))
                except ValueError:
                    continue
                try:
                    watts.append(float(parts[3]))
                except ValueError:
                    pass
                for name, val in zip(names, parts[5:9]):
                    if val.lower() == "active":
                        reasons.add(name)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w": statistics.median(watts) if watts else None}


def cpu_baseline(grid, gens: int):
    """The reference's CAT engine (oracle/_ref, built from the reference sources)
    on the host's cores: run_engine(Cat) over the full torus for `gens`
    generations, layout conversion included as catbench does."""
    import oracle
    ref = oracle.Reference()
    cores = max(1, ref.hardware_concurrency())
    t0 = time.perf_counter()
    ref.run_engine("cat", grid, RULE, gens, workers=cores)
    dt = time.perf_counter() - t0
    n = grid.shape[0]
    return {"value": n * n * gens / dt, "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"{n}x{n} torus, {gens} generations of run_engine(Cat) with "
                      f"workers={cores} (layout conversion included), {dt:.1f} s"}


def reference_arm(args, rank):
    """--impl reference: the reference's own CPU path on this box's host cores."""
    if rank != 0:
        return
    import numpy as np

    import oracle
    ref = oracle.Reference()
    cores = max(1, ref.hardware_concurrency())
    # calibrate: size the per-step sample so K + W steps fit in ~2 minutes
    probe = 1024
    g = ref.init_random(probe, DENSITY, SEED)
    t0 = time.perf_counter()
    ref.run_engine("cat", g, RULE, 2, workers=cores)
    rate = probe * probe * 2 / (time.perf_counter() - t0)
    budget_s = 120.0
    per_step = budget_s / max(1, args.steps + args.warmup)
    n_s = int((rate * per_step) ** 0.5) // 16 * 16
    n_s = max(64, min(N_SIDE, n_s))
    grid = ref.init_random(n_s, DENSITY, SEED)
    if args.warmup:
        grid = ref.run_engine("cat", grid, RULE, args.warmup, workers=cores)
    t0 = time.perf_counter()
    ref.run_engine("cat", grid, RULE, args.steps, workers=cores)
    dt = time.perf_counter() - t0
    value = n_s * n_s * args.steps / dt
    sample = (f"{n_s}x{n_s} torus (bounded sample of the {N_SIDE}^2 workload, same rule and "
              f"density), {args.steps} generations in one run_engine(Cat) call, workers={cores}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (init_random splitmix64 grid, density 0.21, seed 1)",
        "config": {"workload": "configs[1] Bosco r=5 (R5,C2,M1,S34..58,B34..45,NM)",
                   "n": n_s, "rule": RULE, "density": DENSITY, "seed": SEED},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    np.asarray(0)
    print(json.dumps(line), flush=True)


def ours_single(args):
    import numpy as np
    import torch

    from paper_2406_17284_b200 import ltl
    n, steps, warmup = args.n, args.steps, args.warmup
    rule = ltl.parse_ltl_rule(args.rule)
    stencil = args.engine == "stencil"
    torus = ltl.DeviceTorus(rows=n, cols=n)
    torus.init_random(DENSITY, SEED)
    init = torus.download()

    clocks = Clocks()
    clocks.start()
    total_ms, kernel_ms = torus.time(rule, steps, warmup, stencil=stencil)
    launches = torus.time_launches()  # inside the timed loop
    clk = clocks.stop()

    cells = n * n
    value = cells * steps / (total_ms / 1e3)
    kern_avg_s = kernel_ms / 1e3 / steps
    peaks, peak_kind = measured_peaks()
    achieved = BYTES_PER_CELL * cells / kern_avg_s / 1e9
    traffic, traffic_n = ncu_traffic()
    if traffic is not None and traffic_n != n:
        traffic = traffic * (n * n) / (traffic_n * traffic_n)

    # e2e through the public C-ABI: pinned host buffers, run_engine(Cat) semantics
    hin = torch.from_numpy(init).pin_memory().numpy()
    hout = torch.empty((n, n), dtype=torch.uint8).pin_memory().numpy()
    torus.run_interior(hin, rule, 1, out=hout, stencil=stencil)  # warm
    iters = 2
    t0 = time.perf_counter()
    for _ in range(iters):
        torus.run_interior(hin, rule, steps, out=hout, stencil=stencil)
    e2e_s = time.perf_counter() - t0
    e2e_value = cells * steps * iters / e2e_s

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": steps,
        "warmup": warmup, "ms_per_step": total_ms / steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (device init_random, splitmix64 grid identical to the reference's)",
        "config": {"workload": "configs[1] Bosco r=5 16384x16384, 1 generation per step",
                   "rule": args.rule, "n": n, "density": DENSITY, "seed": SEED,
                   "engine": "tcgen05 banded-MMA" if not stencil else "CUDA-core stencil",
                   "l2": "inputs larger than L2 (2 x 256 MiB ping-pong generations)",
                   "parallelism": "1 slab"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": cells,
                "d2h_bytes_per_step": cells,
                "step": f"one ltl_run_interior call = upload + {steps} generations + download"},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                     "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                     "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)",
                     "kernel_ms_per_generation": kern_avg_s * 1e3,
                     "algorithmic_bytes_per_generation": BYTES_PER_CELL * cells,
                     "per": ("generation: one persistent launch runs all timed generations"
                             if launches == 1 and steps > 1 else
                             "generation: one step-kernel launch each")},
        "clocks": clk,
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(init, args.cpu_gens)
    np.asarray(0)
    print(json.dumps(line), flush=True)


def ours_multi(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2406_17284_b200 import ltl
    from paper_2406_17284_b200.dist import PartitionedTorus
    n, steps, warmup = args.n, args.steps, args.warmup
    rule = ltl.parse_ltl_rule(args.rule)
    stencil = args.engine == "stencil"
    torch.cuda.set_device(local_rank)
    part = PartitionedTorus(world * n, n, rank, world, local_rank, ring=not stencil)
    stream = torch.cuda.current_stream()
    part.use_stream(stream.cuda_stream)
    part.init_random(DENSITY, SEED)
    if stencil:
        for _ in range(warmup):
            part.step(rule, stencil)
    else:
        part.run(rule, warmup)
    torch.cuda.synchronize()
    dist.barrier()
    l0 = part.torus.kernel_launches()
    clocks = Clocks() if rank == 0 else None
    if clocks:
        clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    if stencil:
        for _ in range(steps):
            part.step(rule, stencil)
    else:
        part.run(rule, steps)
    ev1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    launches = part.torus.kernel_launches() - l0
    clk = clocks.stop() if clocks else None
    ms = torch.tensor([ev0.elapsed_time(ev1)], device="cuda", dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    total_ms = float(ms.item())
    cells = world * n * n
    value = cells * steps / (total_ms / 1e3)

    # e2e: each rank uploads its slab from pinned memory, runs, downloads
    hin = torch.from_numpy(part.torus.download()).pin_memory().numpy()
    hout = torch.empty_like(torch.from_numpy(hin)).pin_memory().numpy()
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    part.torus.upload(hin)
    part.exchange()
    if stencil:
        for _ in range(steps):
            part.step(rule, stencil)
    else:
        part.run(rule, steps)
    part.torus.download(hout)
    torch.cuda.synchronize()
    e2e = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
    dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    e2e_value = cells * steps / float(e2e.item())
    if rank == 0:
        peaks, peak_kind = measured_peaks()
        achieved = BYTES_PER_CELL * (n * n) / (total_ms / 1e3 / steps) / 1e9
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": warmup, "ms_per_step": total_ms / steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (device init_random, splitmix64 grid identical to the reference's)",
            "config": {"workload": f"configs[1] Bosco r=5, {n}x{n} cells per GPU, "
                                   f"({world}*{n})x{n} torus in row slabs",
                       "rule": args.rule, "n": n, "density": DENSITY, "seed": SEED,
                       "l2": "inputs larger than L2",
                       "parallelism": (f"row slabs x{world}, 16-row halo exchange fused into "
                                       f"the step (TMA stores into the ring neighbours' "
                                       f"halo buffers over NVLink, CUDA IPC)" if part.ring else
                                       f"row slabs x{world}, 16-row NCCL halo exchange")},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": n * n * world,
                    "d2h_bytes_per_step": n * n * world,
                    "step": f"upload + {steps} generations + download per rank"},
            "gpu_launches": launches * world,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                         "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": None,
                         "peak_source": f"{peak_kind} hbm_gbs, per GPU, whole step time"},
            "clocks": clk,
        }
        np.asarray(0)
        print(json.dumps(line), flush=True)


def torch_device(local_rank):
    import torch
    return torch.device("cuda", local_rank)


def main():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--engine", choices=("cat", "stencil"), default="cat")
    ap.add_argument("--n", type=int, default=N_SIDE)
    ap.add_argument("--rule", default=RULE)
    ap.add_argument("--cpu-gens", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist", action="store_true",
                    help="use the multi-process slab path even at world size 1 (testing)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        reference_arm(args, rank)
        return
    if world > 1 or args.dist:
        import torch.distributed as dist
        if "RANK" not in os.environ:  # --dist without torchrun: a world of one
            os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1",
                              MASTER_PORT=os.environ.get("MASTER_PORT", "29533"))
        dist.init_process_group(os.environ.get("LTL_DIST_BACKEND", "nccl"),
                                device_id=torch_device(local_rank))
        try:
            ours_multi(args, rank, world, local_rank)
        finally:
            dist.destroy_process_group()
    else:
        ours_single(args)


if __name__ == "__main__":
    main()
