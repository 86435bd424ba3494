#!/usr/bin/env python
"""bench.py -- cell updates/s of the B200 LTL step (BASELINE.json metric:
"cell updates/sec vs radius r=1..16 at 1/2/4/8 B200; % of roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c1|c2|c3|c4] [--engine cat|base|pack|cat-4bit]

Workloads (BASELINE.json configs; all grids from init_random(n, density,
seed 1), generated on the device bit-identically to the reference's
splitmix64 grid):

  c2  (default at N=1, the config the metric is quoted on) the radius sweep:
      the 16 Table-III presets r = 1..16 (proj/src/rule.cpp:113-133) at their
      densities, each on its own 32768 x 32768 torus.  One bench step = one
      generation of every radius (16 x 2^30 cell updates).  `value` = the
      minimum over r of the per-radius cell updates/s; `per_radius` lists all.
  c4  (default at N>1) weak scaling: r = 8 `globe`, 65536^2 cells per GPU, an
      (N*65536) x 65536 torus in row slabs, halo exchange fused into the step.
  c3  strong scaling: r = 16 `tangy-ramen`, one 65536^2 torus split in N slabs.
  c1  Bosco r=5 (R5,C2,M1,S34..58,B34..45,NM) 16384^2, one generation per step.

`value` is device-timed (CUDA events on the launching stream around the K
timed generations, max over ranks) with the grid resident in HBM; every
generation buffer (>= 1 GiB for c2..c4) exceeds the 126 MB L2, so no flush is
needed.  `e2e` is the same metric through the public C-ABI call a user makes
(ltl_run_interior = run_engine(Cat): upload from pinned host memory, K
generations, download), wall-clocked -- the reference's own bench protocol
(catbench bench times whole run_engine calls, tools/catbench.cpp:123-130).

--impl reference times the reference's own CPU CAT engine (oracle/_ref, the
unmodified reference sources compiled by oracle/Makefile) on this box's host
cores on the same workload: same n, same rules and densities, one generation
of one radius per step (radius 1 + step mod 16).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cell updates/sec vs radius r=1..16 at 1/2/4/8 B200; % of roofline"
UNIT = "cell updates/s"
SEED = 1
BYTES_PER_CELL = 2   # read 1 B state + write 1 B next state
OPS_ALG = 192        # the reference's 6 fragment MMAs x 2*16^3 / 16^2
OPS_EXEC = 800       # tcgen05 kind::i8 ops the kernel issues per cell
OPS_EXEC_WIDE = 960  # the same for the r = 17..32 boxes (6 x M128.N192.K32 + 12 x M128.N64.K32)
OPS_EXEC_4BIT = 880  # 4-bit cells: + one bias MMA (M128.N160.K32 kind::f8f6f4) per 128 x 128 unit
BOSCO = "R5,C2,M1,S34..58,B34..45,NM"

WORKLOADS = {
    "c0": "configs[0] Game of Life (R1,C2,M0,S2..3,B3..3,NM) 1024x1024, density 0.5",
    "c1": "configs[1] Bosco r=5 (R5,C2,M1,S34..58,B34..45,NM) 16384x16384",
    "c2": "configs[2] radius sweep r=1..16 (Table III presets) 32768x32768",
    "c3": "configs[3] r=16 tangy-ramen 65536x65536 row slabs (strong scaling)",
    "c4": "configs[4] r=8 globe 65536x65536 cells per GPU (weak scaling)",
    "wide": "extension: radius sweep r=17..32 (majority rules) 32768x32768 (PAPER.md:561)",
}


def majority_rule(r):
    """Majority rule at radius r (the shape of the r=4 preset `majority`,
    S40..80 B41..80): survive with >= half, born with > half of the
    (2r+1)^2 - 1 neighbours alive; density 0.5."""
    cells = (2 * r + 1) ** 2 - 1
    return f"R{r},C2,M0,S{cells // 2}..{cells},B{cells // 2 + 1}..{cells},NM"


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured (MEASURED_PEAKS.json)"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback (B200_PROFILING.md)"


def profile_json(name):
    try:
        with open(os.path.join(ROOT, "profiles", name)) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return None


def mma_i8_peak():
    """Measured tcgen05 kind::i8 dense peak (tools/ubench_mma.cu on a B200,
    profiles/ubench_mma_r02.json), else the vendor figure."""
    d = profile_json("ubench_mma_r02.json")
    if d and d.get("i8_peak_tops"):
        return float(d["i8_peak_tops"]) * 1e12, "measured (profiles/ubench_mma_r02.json)"
    return 4.5e15, "vendor dense i8 (no measurement committed)"


def workload_rules(workload):
    """[(label, rule text, density)] of a workload (the reference's presets)."""
    from paper_2406_17284_b200 import ltl
    presets = ltl.ltl_presets()
    if workload == "c0":
        return [("life", presets[0][1], 0.5)]
    if workload == "c1":
        return [("bosco-literal", BOSCO, 0.21)]
    if workload == "c2":
        return [(p[0], p[1], p[2]) for p in presets[:16]]
    if workload == "c3":
        return [tuple(presets[15])]
    if workload == "wide":
        return [(f"majority-r{r}", majority_rule(r), 0.5) for r in range(17, 33)]
    return [tuple(presets[7])]


def workload_side(workload):
    return {"c0": 1024, "c1": 16384, "c2": 32768, "c3": 65536, "c4": 65536, "wide": 32768}[workload]


class Clocks:
    """SM clock / throttle sampler running during the timed region: NVML every
    20 ms (nvidia_ml_py; light enough not to disturb the timed launches), else
    nvidia-smi every 100 ms."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, device=0):
        self.device = device
        self.samples, self.reasons, self.watts, self.max_mhz = [], set(), [], 0
        self.stop_ev = threading.Event()
        self.thread = None
        self.proc = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def loop():
                while not self.stop_ev.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        mask = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for k, bit in self.REASONS.items():
                            if mask & bit:
                                self.reasons.add(k)
                        self.watts.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0)
                    except Exception:  # noqa: BLE001
                        pass
                    time.sleep(0.020)
            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
            return
        except Exception:  # noqa: BLE001 -- no NVML: nvidia-smi
            pass
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.thread:
            self.stop_ev.set()
            self.thread.join()
        elif self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            self.proc.wait()
            with open(self.path) as fh:
                for line in fh:
                    parts = [p.strip() for p in line.split(",")]
                    try:
                        self.samples.append(float(parts[0]))
                        self.max_mhz = max(self.max_mhz, float(parts[1]))
                        self.watts.append(float(parts[2]))
                    except (ValueError, IndexError):
                        continue
                    for k, v in zip(list(self.REASONS), parts[3:7]):
                        if v.lower() == "active":
                            self.reasons.add(k)
            os.unlink(self.path)
        if not self.samples:
            return None
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "power_w": statistics.median(self.watts) if self.watts else None}


# --------------------------------------------------------------------- CPU legs
def cpu_baseline(grids, rules, n):
    """The reference's CPU CAT engine (oracle/_ref) on this box's host cores,
    one generation of each sampled radius: run_engine(Cat) with the layout
    conversion (catbench style) and simulate() alone."""
    import oracle
    ref = oracle.Reference()
    cores = max(1, ref.hardware_concurrency())
    tot_ms = sim_ms = 0.0
    for g, (label, rule, _d) in zip(grids, rules):
        a, b = ref.run_cat_timed(g, rule, 1, workers=cores)
        tot_ms += a
        sim_ms += b
    gens = len(grids)
    labels = ",".join(r[0] for r in rules)
    return {"value": n * n * gens / (tot_ms / 1e3), "unit": UNIT, "cores": cores,
            "kind": "reference",
            "value_simulate_only": n * n * gens / (sim_ms / 1e3),
            "sample": f"{n}x{n} torus, 1 generation each of {labels} through run_engine(Cat) "
                      f"with workers={cores}: {tot_ms / 1e3:.1f} s with the layout conversion "
                      f"(value), {sim_ms / 1e3:.1f} s in simulate() alone (value_simulate_only)"}


def reference_arm(args, rank, world):
    """--impl reference: the reference's own CPU path on this box's host cores."""
    if rank != 0:
        return
    if args.workload == "wide":
        print(json.dumps({"impl": "reference", "unavailable": "the reference's engines reject "
                          "r > 16 (proj/src/rule.cpp:33-35)"}), flush=True)
        return
    import numpy as np

    import oracle
    ref = oracle.Reference()
    cores = max(1, ref.hardware_concurrency())
    workload = args.workload
    rules = ref_rules(ref, workload)
    n = workload_side(workload)
    note = ""
    if workload in ("c3", "c4"):
        # one 65536^2 CAT step needs ~56 GB of host RAM and ~1 min per
        # generation on 16 cores: bounded sample of the same rule at 16384^2
        n = 16384
        note = f" (bounded sample: {n}^2 torus of the same rule; the GPU arm's torus is " \
               f"{'N*' if workload == 'c4' else ''}65536 x 65536)"
    else:
        # each step a bounded sample so the whole run ends within minutes: the
        # reference CAT engine does ~5.5e7 cell updates/s on 16 cores, flat in
        # n and r (profiles/bench_ref_c2_r02a.json: 19.4 s per 32768^2
        # generation); the largest square torus whose W + K generations fit
        # in ~5 min
        full = n
        while n > 4096 and (args.warmup + args.steps) * n * n / 5.5e7 > 300:
            n //= 2
        if n != full:
            note = (f" (bounded sample: {n}^2 torus of the same rules and densities, so that the "
                    f"{args.warmup} + {args.steps} generations end within minutes; the GPU arm's "
                    f"torus is {full} x {full})")
    # the initial grids, built by the reference's init_random in parallel threads
    grids = [None] * len(rules)

    def mk(i):
        grids[i] = ref.init_random(n, rules[i][2], SEED)
    ths = [threading.Thread(target=mk, args=(i,)) for i in range(len(rules))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    per = {}
    total = 0.0
    for i in range(args.warmup + args.steps):
        k = i % len(rules)
        t0 = time.perf_counter()
        grids[k] = ref.run_engine("cat", grids[k], rules[k][1], 1, workers=cores)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            total += dt
            per.setdefault(k, []).append(dt)
    rates = {k: n * n * len(v) / sum(v) for k, v in per.items()}
    value = min(rates.values())
    sample = (f"{n}x{n} torus{note}; step i = one generation of radius "
              f"{'1 + i mod 16' if len(rules) > 1 else rules[0][0]} through run_engine(Cat) "
              f"(layout conversion included, as catbench), workers={cores}; value = min over "
              f"the radii timed of their cell updates/s")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak" if workload != "c3" else "strong",
        "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (reference init_random splitmix64 grids, seed 1)",
        "config": config_dict(workload, world),
        "aggregate_value": n * n * args.steps / total,
        "per_radius": [{"r": ref.parse_rule(rules[k][1])[0], "rule": rules[k][0],
                        "cell_updates_per_s": rates[k], "generations": len(per[k])}
                       for k in sorted(per)],
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    np.asarray(0)
    print(json.dumps(line), flush=True)


def ref_rules(ref, workload):
    presets = ref.presets()
    if workload == "c0":
        return [("life", presets[0][1], 0.5)]
    if workload == "c1":
        return [("bosco-literal", BOSCO, 0.21)]
    if workload == "c2":
        return [tuple(p) for p in presets[:16]]
    if workload == "c3":
        return [tuple(presets[15])]
    if workload == "wide":
        return [(f"majority-r{r}", majority_rule(r), 0.5) for r in range(17, 33)]
    return [tuple(presets[7])]


def config_dict(workload, world):
    n = workload_side(workload)
    d = {"workload": WORKLOADS[workload], "n": n, "seed": SEED,
         "l2": "inputs larger than L2 (every generation buffer >= 256 MiB > 126 MB L2)"}
    if workload == "c2":
        d["rules"] = "Table III presets r=1..16 at their densities (proj/src/rule.cpp:113-133)"
    elif workload == "wide":
        d["rules"] = ("majority rules r=17..32 at density 0.5 (the reference's engines reject "
                      "r > 16; parity: tests/test_gpu_wide.py)")
    elif workload == "c1":
        d.update(rule=BOSCO, density=0.21)
    elif workload == "c0":
        d.update(rule="R1,C2,M0,S2..3,B3..3,NM", density=0.5,
                 l2="L2-resident (2 x 1.1 MB): launch / latency bound, no HBM roofline")
    elif workload == "c3":
        d.update(rule="R16,C2,M0,S170..296,B170..300,NM", density=0.26,
                 torus=f"{n}x{n} split in {world} row slabs")
    else:
        d.update(rule="R8,C2,M0,S163..223,B74..252,NM", density=0.23,
                 torus=f"({world}*{n})x{n} in {world} row slabs")
    d["parallelism"] = ("1 slab" if world == 1 else
                        f"row slabs x{world}, 16-row halo pulled by the step's own TMA loads "
                        f"from the ring neighbours' slabs over NVLink (CUDA IPC)")
    return d


# --------------------------------------------------------------------- GPU arm
def ours_single(args):
    import numpy as np
    import torch

    from paper_2406_17284_b200 import ltl
    workload, steps, warmup = args.workload, args.steps, args.warmup
    n = workload_side(workload)
    rules = workload_rules(workload)
    engine = args.engine
    mma_engine = engine in ("cat", "cat-4bit")
    # algorithmic bytes per cell update: u8 cells 2 (read + write), 4-bit cells 1
    bpc = 1 if engine == "cat-4bit" else BYTES_PER_CELL
    torus = ltl.DeviceTorus(rows=n, cols=n)

    clocks = Clocks(torch.cuda.current_device())
    per, launches, inits = [], 0, []
    clocks.start()
    for label, rule_text, dens in rules:
        rule = ltl.parse_ltl_rule(rule_text, max_radius=ltl.MAX_WIDE_RADIUS)
        torus.init_random(dens, SEED)
        if workload == "c2" and label in ("life", "bosco", "tangy-ramen"):
            inits.append((label, rule_text, dens, torus.download()))
        total_ms, kernel_ms = torus.time(rule, steps, warmup, engine=engine)
        launches += torus.time_launches()
        per.append(dict(r=rule.r, rule=label, ms_per_generation=total_ms / steps,
                        kernel_ms_isolated=kernel_ms / steps,
                        cell_updates_per_s=n * n * steps / (total_ms / 1e3)))
    clk = clocks.stop()

    peaks, peak_src = measured_peaks()
    hbm = peaks["hbm_gbs"]
    p_mma, mma_src = mma_i8_peak()
    for e in per:
        e["hbm_frac"] = bpc * n * n / (e["ms_per_generation"] / 1e3) / 1e9 / hbm
    ms_step = sum(e["ms_per_generation"] for e in per)
    value = min(e["cell_updates_per_s"] for e in per)
    # The timed region launches the step kernel only (gpu_launches = one per
    # generation and radius), back to back on one stream: its average launch
    # duration is the region's event time / launches.  (Bracketing every launch
    # with its own events -- kernel_ms_isolated -- cuts the programmatic overlap
    # of consecutive launches and reads ~4 % longer.)
    kern_avg_s = statistics.mean(e["ms_per_generation"] for e in per) / 1e3
    kern_iso_s = statistics.mean(e["kernel_ms_isolated"] for e in per) / 1e3
    achieved = bpc * n * n / kern_avg_s / 1e9
    ceiling_hbm = hbm * 1e9 / bpc
    ops_exec = (OPS_EXEC_WIDE if workload == "wide" else
                OPS_EXEC_4BIT if engine == "cat-4bit" else OPS_EXEC)
    ceiling_mma = p_mma / ops_exec if mma_engine else None

    # e2e through the public C-ABI (ltl_run_interior = run_engine(Cat)):
    # pinned host grids, upload + K generations + download per radius
    hin = torch.empty((n, n), dtype=torch.uint8).pin_memory().numpy()
    hout = torch.empty((n, n), dtype=torch.uint8).pin_memory().numpy()
    e2e_s, e2e_per, moved = 0.0, [], [0, 0]
    for label, rule_text, dens in rules:
        rule = ltl.parse_ltl_rule(rule_text, max_radius=ltl.MAX_WIDE_RADIUS)
        torus.init_random(dens, SEED)
        torus.download(hin)
        torus.run_interior(hin, rule, 1, out=hout, engine=engine)  # warm
        b0 = torus.transfer_bytes()
        t0 = time.perf_counter()
        torus.run_interior(hin, rule, steps, out=hout, engine=engine)
        dt = time.perf_counter() - t0
        b1 = torus.transfer_bytes()
        moved = [moved[0] + b1[0] - b0[0], moved[1] + b1[1] - b0[1]]
        e2e_s += dt
        e2e_per.append(n * n * steps / dt)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": steps,
        "warmup": warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (device init_random, splitmix64 grids identical to the reference's)",
        "config": dict(config_dict(workload, 1),
                       engine={"cat": "tcgen05 banded-MMA", "base": "CUDA-core direct-sum stencil",
                               "pack": "CUDA-core packed sliding-window stencil",
                               "cat-4bit": "tcgen05 banded-MMA on 4-bit device cells "
                                           "(pass 1 kind::f8f6f4 e4m3 x e2m1)"}[engine],
                       step=(f"one generation of each of the {len(rules)} radii"
                             if len(rules) > 1 else "one generation")),
        "aggregate_value": n * n * len(rules) / (ms_step / 1e3),
        "per_radius": per,
        "e2e": {"value": min(e2e_per), "unit": UNIT,
                "h2d_bytes_per_step": moved[0] // steps,
                "d2h_bytes_per_step": moved[1] // steps,
                "step": (f"per radius one ltl_run_interior call (run_engine(Cat)): the {n}x{n} "
                         f"u8 grid from pinned host memory to the device (bit-packed on the host "
                         f"cores in flight: one bit per cell over PCIe), {steps} generations, back "
                         f"into pinned host memory the same way; value = min over r; bytes = "
                         f"ltl_transfer_bytes, amortised over the call's {steps} generations"),
                "aggregate_value": n * n * steps * len(rules) / e2e_s},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": None, "peak_source": peak_src,
                     "kernel": "ltl_tc_step_kernel" if mma_engine else f"{engine} stencil",
                     "kernel_ms_per_generation": kern_avg_s * 1e3,
                     "kernel_ms_isolated": kern_iso_s * 1e3,
                     "algorithmic_bytes_per_generation": bpc * n * n,
                     "per": ("generation: timed-region event time / launches (one step-kernel "
                             "launch per generation), mean over the radii"),
                     "ceiling_cells_per_s_hbm": ceiling_hbm,
                     "ceiling_cells_per_s_mma": ceiling_mma,
                     "mma_peak_ops": p_mma if mma_engine else None,
                     "mma_peak_source": mma_src if mma_engine else None,
                     "ops_per_cell_algorithmic": OPS_ALG, "ops_per_cell_executed":
                         ops_exec if mma_engine else None,
                     "mma_frac": (value * ops_exec / p_mma) if mma_engine else None},
        "clocks": clk,
    }
    ncu_name = f"ncu_tc_step_{'wide_' if workload == 'wide' else ''}{n}.json"
    ncu = profile_json(ncu_name)
    if ncu and engine == "cat":
        line["roofline"]["traffic"] = ncu.get("dram_bytes_per_generation")
        line["roofline"]["traffic_source"] = f"profiles/{ncu_name} (ncu --set full)"
    if not args.no_cpu_baseline and inits:
        line["cpu_baseline"] = cpu_baseline([g for *_, g in inits],
                                            [(a, b, c) for a, b, c, _ in inits], n)
    np.asarray(0)
    print(json.dumps(line), flush=True)


def ours_multi(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2406_17284_b200 import ltl
    from paper_2406_17284_b200.dist import PartitionedTorus
    workload, steps, warmup = args.workload, args.steps, args.warmup
    n = workload_side(workload)
    label, rule_text, dens = workload_rules(workload)[0]
    rule = ltl.parse_ltl_rule(rule_text)
    dev = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    cdev = "cuda" if dist.get_backend() == "nccl" else "cpu"  # where collective tensors live
    global_rows = n if workload == "c3" else world * n
    part = PartitionedTorus(global_rows, n, rank, world, dev)
    stream = torch.cuda.current_stream()
    part.use_stream(stream.cuda_stream)
    part.init_random(dens, SEED)
    part.run(rule, warmup)
    torch.cuda.synchronize()
    dist.barrier()
    l0 = part.torus.kernel_launches()
    clocks = Clocks(dev) if rank == 0 else None
    if clocks:
        clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    part.run(rule, steps)
    ev1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    launches = torch.tensor([part.torus.kernel_launches() - l0], device=cdev)
    dist.all_reduce(launches)
    clk = clocks.stop() if clocks else None
    ms = torch.tensor([ev0.elapsed_time(ev1)], device=cdev, dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    total_ms = float(ms.item())
    cells = global_rows * n
    value = cells * steps / (total_ms / 1e3)

    # e2e: each rank uploads its slab from pinned memory, runs, downloads
    hin = torch.from_numpy(part.torus.download()).pin_memory().numpy()
    hout = torch.empty_like(torch.from_numpy(hin)).pin_memory().numpy()
    torch.cuda.synchronize()
    dist.barrier()
    b0 = part.torus.transfer_bytes()
    t0 = time.perf_counter()
    part.upload(hin)
    part.run(rule, steps)
    part.torus.download(hout)
    torch.cuda.synchronize()
    e2e = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=cdev)
    dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    b1 = part.torus.transfer_bytes()
    moved = torch.tensor([b1[0] - b0[0], b1[1] - b0[1]], dtype=torch.int64, device=cdev)
    dist.all_reduce(moved)  # all ranks' bytes
    e2e_value = cells * steps / float(e2e.item())
    parity = g_vs_1_check(part, hout, rule, dens, warmup + 2 * steps, global_rows, n, rank, world)
    if rank == 0:
        peaks, peak_src = measured_peaks()
        hbm = peaks["hbm_gbs"]
        achieved = BYTES_PER_CELL * part.rows * n / (total_ms / 1e3 / steps) / 1e9
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": warmup, "ms_per_step": total_ms / steps, "higher_is_better": True,
            "scaling": "strong" if workload == "c3" else "weak", "vs_baseline": None,
            "dtype": "u8",
            "data": "synthetic (device init_random, splitmix64 grid identical to the reference's)",
            "config": dict(config_dict(workload, world), rule_name=label,
                           exchange="fused ring pulls" if part.ring else "NCCL send/recv"),
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": int(moved[0].item()) // steps,
                    "d2h_bytes_per_step": int(moved[1].item()) // steps,
                    "step": f"upload + {steps} generations + download per rank (bit-packed "
                            f"PCIe transfers); bytes = all ranks' ltl_transfer_bytes, amortised "
                            f"over the {steps} generations"},
            "gpu_launches": int(launches.item()),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": None, "peak_source": peak_src,
                         "per": "generation per GPU (rank 0's slab, whole step time)"},
            "clocks": clk,
            "parity": parity,
        }
        ncu = profile_json(f"ncu_tc_step_{n}.json")
        if ncu:
            line["roofline"]["traffic"] = ncu.get("dram_bytes_per_generation")
            line["roofline"]["traffic_source"] = (f"profiles/ncu_tc_step_{n}.json (1-GPU "
                                                  f"{n}^2 capture, per {n}^2 generation)")
        if not args.no_cpu_baseline:
            import oracle
            ref = oracle.Reference()
            g = ref.init_random(4096, dens, SEED)
            line["cpu_baseline"] = cpu_baseline([g], [(label, rule_text, dens)], 4096)
            line["cpu_baseline"]["sample"] += " (4096^2 bounded sample of the same rule)"
        np.asarray(0)
        print(json.dumps(line), flush=True)


def g_vs_1_check(part, slab, rule, dens, gens, global_rows, n, rank, world):
    """Bit-exactness of the G-GPU run: every rank's final slab (CRC-32 +
    alive count) against the same torus run for the same generations on ONE
    GPU by rank 0 (after the timed region; device init is bit-identical, so
    both start from the same grid)."""
    import zlib

    import numpy as np
    import torch.distributed as dist

    from paper_2406_17284_b200 import ltl
    mine = (part.row0, part.rows, zlib.crc32(memoryview(np.ascontiguousarray(slab))),
            int(np.count_nonzero(slab)))
    table = [None] * world
    dist.all_gather_object(table, mine)
    ok = None
    if rank == 0:
        with ltl.DeviceTorus(rows=global_rows, cols=n) as t:
            t.init_random(dens, SEED)
            t.run(rule, gens)
            full = t.download()
        from concurrent.futures import ThreadPoolExecutor

        def same(entry):  # zlib / numpy release the GIL: slabs checked in parallel
            r0, rows, crc, alive = entry
            part_rows = full[r0:r0 + rows]
            return (zlib.crc32(memoryview(part_rows)) == crc and
                    int(np.count_nonzero(part_rows)) == alive)
        with ThreadPoolExecutor(max_workers=min(8, world)) as pool:
            ok = all(pool.map(same, table))
    dist.barrier()
    return {"g_vs_1_bit_exact": ok, "generations": gens,
            "how": f"each rank's slab after {gens} generations (CRC-32 + alive count) vs the "
                   f"{global_rows}x{n} torus run on one GPU by rank 0"}


def spawn(args):
    """--gpus N without a torchrun environment: re-launch under torchrun."""
    port = os.environ.get("MASTER_PORT", str(29500 + os.getpid() % 1000))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=tuple(WORKLOADS), default=None)
    ap.add_argument("--engine", choices=("cat", "base", "pack", "cat-4bit"), default="cat")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist", action="store_true",
                    help="the multi-process slab path even at world size 1 (testing)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        if args.impl == "reference":
            world = args.gpus  # rank 0 alone runs the CPU reference
        else:
            spawn(args)
    if args.workload is None:
        args.workload = "c2" if max(world, args.gpus) == 1 else "c4"
    if args.impl == "reference":
        reference_arm(args, rank, max(world, args.gpus))
        return
    if world > 1 or args.dist:
        import torch
        import torch.distributed as dist
        if "RANK" not in os.environ:  # --dist without torchrun: a world of one
            os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1",
                              MASTER_PORT=os.environ.get("MASTER_PORT", "29533"))
        # one rank per GPU over NCCL; more ranks than GPUs (a smoke run of the
        # multi-process path on a small box): ranks share GPUs, the control
        # collectives go over gloo (the slabs' rows move over CUDA IPC either way)
        ndev = max(1, torch.cuda.device_count())
        if world <= ndev:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")
        try:
            ours_multi(args, rank, world, local_rank)
        finally:
            dist.destroy_process_group()
    else:
        ours_single(args)


if __name__ == "__main__":
    main()
