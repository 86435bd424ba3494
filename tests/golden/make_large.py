"""Large-size parity fixtures for BASELINE.json configs[1..4], produced by the
UNMODIFIED reference (oracle/_ref) at the sizes the configs state.

Run here (the container that has /root/reference), one config per process so
they can share the cores:

    make -C oracle
    python tests/golden/make_large.py c2 --workers 4     # 32768^2, r=1..16, 2 steps  (~10 min)
    python tests/golden/make_large.py c1 --workers 6     # 16384^2 Bosco, 1000 steps  (~1 h)
    python tests/golden/make_large.py c3                 # 65536^2 r=16, 2 steps, BASE (~25 min)
    python tests/golden/make_large.py c4                 # 65536^2 r=8,  2 steps, BASE (~10 min)

Each writes tests/golden/large_<cfg>.json incrementally.  The grids are never
stored: every entry records the alive count, the FNV-1a-64 of the n*n
row-major interior and the FNV of each of 16 equal row blocks (to localise a
mismatch), for the initial grid (init_random, seed 1: the GPU tests rebuild it
with the device init) and after the listed generation counts.

Engines: the reference's CAT engine (run_engine(Cat), workers threads) where
its per-step H/R IntFields fit in host RAM (configs 1-2); the reference's BASE
engine (simulate_base, the reference's own oracle, single-threaded) at 65536^2,
where CAT's two 17.2 GB IntFields per step would not (SURVEY.md §7 "verification
cost at scale").  Both are the reference's code, verified equal by its own
acceptance criterion 1.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
BLOCKS = 16

BOSCO_LITERAL = "R5,C2,M1,S34..58,B34..45,NM"   # BASELINE configs[1]


def digest(orc: oracle.Oracle, g: np.ndarray) -> dict:
    n = g.shape[0]
    rb = n // BLOCKS
    return dict(alive=int(np.count_nonzero(g)),
                fnv=f"{orc.fnv1a64(g):016x}",
                block_rows=rb,
                block_fnv=[f"{orc.fnv1a64(g[i * rb:(i + 1) * rb]):016x}" for i in range(BLOCKS)])


class Sink:
    def __init__(self, name: str, meta: dict):
        self.path = os.path.join(HERE, f"large_{name}.json")
        self.doc = dict(meta, generator="tests/golden/make_large.py (reference oracle/_ref)",
                        hash="FNV-1a-64 over the n*n row-major interior bytes; block_fnv over "
                             "16 equal row blocks", entries=[])
        if os.path.exists(self.path):
            with open(self.path) as fh:
                old = json.load(fh)
            self.doc["entries"] = old.get("entries", [])

    def have(self, key: dict) -> dict | None:
        for e in self.doc["entries"]:
            if all(e.get(k) == v for k, v in key.items()):
                return e
        return None

    def add(self, entry: dict) -> None:
        self.doc["entries"].append(entry)
        with open(self.path + ".tmp", "w") as fh:
            json.dump(self.doc, fh, indent=1)
        os.replace(self.path + ".tmp", self.path)


def run_series(ref, orc, sink, engine, rule, n, dens, checkpoints, workers, tag):
    """init_random(n, dens, 1) then run_engine(engine) up to each checkpoint."""
    key = dict(rule=rule, n=n, density=dens, seed=1)
    if all(sink.have(dict(key, steps=s)) for s in [0] + checkpoints):
        print(f"{tag}: cached", flush=True)
        return
    t0 = time.time()
    g = ref.init_random(n, dens, 1)
    if not sink.have(dict(key, steps=0)):
        sink.add(dict(key, steps=0, engine="init_random", **digest(orc, g)))
    print(f"{tag}: init {time.time() - t0:.1f}s", flush=True)
    done = 0
    for s in checkpoints:
        t1 = time.time()
        g = ref.run_engine(engine, g, rule, s - done, workers=workers)
        done = s
        if not sink.have(dict(key, steps=s)):
            sink.add(dict(key, steps=s, engine=engine, seconds=round(time.time() - t1, 1),
                          **digest(orc, g)))
        print(f"{tag}: steps {s} alive {int(np.count_nonzero(g))} ({time.time() - t1:.1f}s)",
              flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["c1", "c2", "c3", "c4"])
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    a = ap.parse_args()
    ref = oracle.Reference()
    orc = oracle.Oracle()
    presets = ref.presets()
    if a.config == "c1":
        sink = Sink("c1", dict(config="BASELINE configs[1]: Bosco r=5 (literal rule) "
                                      "16384^2, 1000 steps"))
        run_series(ref, orc, sink, "cat", BOSCO_LITERAL, 16384, 0.21, [1, 10, 100, 1000],
                   a.workers, "c1")
    elif a.config == "c2":
        sink = Sink("c2", dict(config="BASELINE configs[2]: radius sweep r=1..16 "
                                      "(Table III presets at their densities) 32768^2"))
        for r in range(1, 17):
            name, rule, dens = presets[r - 1]
            run_series(ref, orc, sink, "cat", rule, 32768, dens, [1, 2], a.workers,
                       f"c2 r={r} {name}")
    elif a.config == "c3":
        name, rule, dens = presets[15]
        sink = Sink("c3", dict(config=f"BASELINE configs[3]: r=16 ({name}) 65536^2"))
        run_series(ref, orc, sink, "base", rule, 65536, dens, [1, 2], 1, "c3")
    else:
        name, rule, dens = presets[7]
        sink = Sink("c4", dict(config=f"BASELINE configs[4]: r=8 ({name}) 65536^2 per GPU "
                                      "(the 1-GPU square torus)"))
        run_series(ref, orc, sink, "base", rule, 65536, dens, [1, 2], 1, "c4")


if __name__ == "__main__":
    main()
