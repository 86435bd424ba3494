"""ctypes front end for the TEST-ONLY checkers in oracle/.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package, and only to check or to time the reference on
the CPU.  The product (paper_2406_17284_b200 + its CUDA library) never does.

* ``Oracle``    -- the C restatement (ltl_oracle.c), built into _build/.
* ``Reference`` -- the unmodified reference library compiled from
                   /root/reference/proj/src (oracle/_ref/libcatsim_ref.so).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libltl_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcatsim_ref.so")

_u8p = ctypes.POINTER(ctypes.c_uint8)
_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u64p = ctypes.POINTER(ctypes.c_uint64)


def build(quiet: bool = True) -> None:
    """make -C oracle (C restatement always; the reference where present)."""
    subprocess.run(["make", "-C", HERE, "-j8"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


class orc_rule(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int32) for k in ("r", "c", "m", "s1", "s2", "b1", "b2", "kind")]

    @classmethod
    def from_ints(cls, v):
        return cls(*[int(x) for x in v])


class Oracle:
    """The plain-C restatement (pinned against the reference by tests/test_oracle.py)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        lib = ctypes.CDLL(path)
        lib.orc_splitmix64_next.argtypes = [_u64p]
        lib.orc_splitmix64_next.restype = ctypes.c_uint64
        lib.orc_alive_threshold.argtypes = [ctypes.c_uint64, ctypes.c_double]
        lib.orc_init_random.argtypes = [ctypes.c_int32, ctypes.c_double, ctypes.c_uint64,
                                        ctypes.c_int32, _u8p]
        lib.orc_apply_transition.argtypes = [ctypes.c_int, ctypes.c_int,
                                             ctypes.POINTER(orc_rule), ctypes.c_int]
        lib.orc_step.argtypes = [_u8p, _u8p, ctypes.c_int32, ctypes.c_int32,
                                 ctypes.POINTER(orc_rule)]
        lib.orc_simulate.argtypes = [_u8p, _u8p, ctypes.c_int32, ctypes.c_int32,
                                     ctypes.POINTER(orc_rule), ctypes.c_int32]
        lib.orc_reductions.argtypes = [_u8p, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.POINTER(orc_rule), _i32p, _i32p]
        lib.orc_fnv1a64.argtypes = [_u8p, ctypes.c_uint64]
        lib.orc_fnv1a64.restype = ctypes.c_uint64
        lib.orc_fill_periodic_halo.argtypes = [_u8p, ctypes.c_int32, ctypes.c_int32]
        self.lib = lib

    def splitmix(self, seed: int, count: int):
        st = ctypes.c_uint64(seed)
        return [self.lib.orc_splitmix64_next(ctypes.byref(st)) for _ in range(count)]

    def alive_threshold(self, z: int, density: float) -> bool:
        return bool(self.lib.orc_alive_threshold(z, density))

    def init_random(self, n: int, density: float, seed: int, fill_n: int = -1) -> np.ndarray:
        out = np.zeros((n, n), np.uint8)
        if self.lib.orc_init_random(n, density, seed, fill_n, _ptr(out, _u8p)) != 0:
            raise ValueError("init_random: invalid arguments")
        return out

    def step(self, grid: np.ndarray, rule) -> np.ndarray:
        g = np.ascontiguousarray(grid, np.uint8)
        out = np.empty_like(g)
        rr = orc_rule.from_ints(rule)
        if self.lib.orc_step(_ptr(g, _u8p), _ptr(out, _u8p), g.shape[0], g.shape[1],
                             ctypes.byref(rr)) != 0:
            raise RuntimeError("internal consistency: negative neighborhood count")
        return out

    def simulate(self, grid: np.ndarray, rule, steps: int) -> np.ndarray:
        g = np.ascontiguousarray(grid, np.uint8)
        out = np.empty_like(g)
        rr = orc_rule.from_ints(rule)
        if self.lib.orc_simulate(_ptr(g, _u8p), _ptr(out, _u8p), g.shape[0], g.shape[1],
                                 ctypes.byref(rr), steps) != 0:
            raise RuntimeError("internal consistency: negative neighborhood count")
        return out

    def reductions(self, grid: np.ndarray, rule):
        g = np.ascontiguousarray(grid, np.uint8)
        h = np.empty(g.shape, np.int32)
        red = np.empty(g.shape, np.int32)
        rr = orc_rule.from_ints(rule)
        self.lib.orc_reductions(_ptr(g, _u8p), g.shape[0], g.shape[1], ctypes.byref(rr),
                                _ptr(h, _i32p), _ptr(red, _i32p))
        return h, red

    def fnv1a64(self, data: np.ndarray) -> int:
        d = np.ascontiguousarray(data, np.uint8)
        return int(self.lib.orc_fnv1a64(_ptr(d, _u8p), d.size))

    def fill_periodic_halo(self, padded: np.ndarray, n: int, halo: int) -> np.ndarray:
        p = np.ascontiguousarray(padded, np.uint8).copy()
        self.lib.orc_fill_periodic_halo(_ptr(p, _u8p), n, halo)
        return p


class ReferenceError_(Exception):
    pass


class Reference:
    """The unmodified reference library (oracle/_ref), C entry points from ref_shim.cpp."""

    ENGINE = {"cat": 0, "base": 1, "pack": 2}

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing (reference not built)")
        lib = ctypes.CDLL(path)
        lib.ref_last_error.restype = ctypes.c_char_p
        lib.ref_splitmix.argtypes = [ctypes.c_uint64, ctypes.c_int32, _u64p]
        lib.ref_alive_threshold.argtypes = [ctypes.c_uint64, ctypes.c_double]
        lib.ref_init_random.argtypes = [ctypes.c_int32, ctypes.c_double, ctypes.c_uint64,
                                        ctypes.c_int32, ctypes.c_int32, _u8p]
        lib.ref_parse_rule.argtypes = [ctypes.c_char_p, _i32p]
        lib.ref_preset.argtypes = [ctypes.c_int32, ctypes.POINTER(ctypes.c_char_p),
                                   ctypes.POINTER(ctypes.c_char_p),
                                   ctypes.POINTER(ctypes.c_double)]
        lib.ref_von_neumann_probe_rule.argtypes = [ctypes.c_int32, _i32p]
        lib.ref_run_engine.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _u8p,
                                       ctypes.c_char_p, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                       _u8p, _i64p]
        lib.ref_reductions.argtypes = [ctypes.c_int32, ctypes.c_int32, _u8p, ctypes.c_char_p,
                                       _i32p, _i32p]
        lib.ref_run_cat_timed.argtypes = [ctypes.c_int32, ctypes.c_int32, _u8p, ctypes.c_char_p,
                                          ctypes.c_int32, ctypes.c_int32, _u8p,
                                          ctypes.POINTER(ctypes.c_double)]
        lib.ref_snapshot_write.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _u8p,
                                           ctypes.c_char_p]
        lib.ref_snapshot_read.argtypes = [ctypes.c_char_p, _i32p, _i32p, _i32p, _u8p,
                                          ctypes.c_int64]
        lib.ref_semantic_steps.argtypes = [ctypes.c_int32, _u8p, _i32p, ctypes.c_int32, _u8p]
        self.lib = lib

    def _check(self, status: int):
        if status != 0:
            msg = self.lib.ref_last_error().decode()
            kind = {1: ValueError, 2: RuntimeError}.get(status, ReferenceError_)
            raise kind(msg)

    def hardware_concurrency(self) -> int:
        return int(self.lib.ref_hardware_concurrency())

    def splitmix(self, seed: int, count: int):
        out = np.zeros(count, np.uint64)
        self.lib.ref_splitmix(seed, count, _ptr(out, _u64p))
        return [int(v) for v in out]

    def alive_threshold(self, z: int, density: float) -> bool:
        return bool(self.lib.ref_alive_threshold(z, density))

    def init_random(self, n: int, density: float, seed: int, f: int = 16,
                    fill_n: int = -1) -> np.ndarray:
        out = np.zeros((n, n), np.uint8)
        self._check(self.lib.ref_init_random(n, density, seed, f, fill_n, _ptr(out, _u8p)))
        return out

    def parse_rule(self, text: str):
        out = np.zeros(8, np.int32)
        self._check(self.lib.ref_parse_rule(text.encode(), _ptr(out, _i32p)))
        return [int(v) for v in out]

    def presets(self):
        res = []
        for i in range(self.lib.ref_preset_count()):
            name, rule, dens = ctypes.c_char_p(), ctypes.c_char_p(), ctypes.c_double()
            self.lib.ref_preset(i, ctypes.byref(name), ctypes.byref(rule), ctypes.byref(dens))
            res.append((name.value.decode(), rule.value.decode(), dens.value))
        return res

    def von_neumann_probe_rule(self, r: int):
        out = np.zeros(8, np.int32)
        self.lib.ref_von_neumann_probe_rule(r, _ptr(out, _i32p))
        return [int(v) for v in out]

    def run_engine(self, engine: str, grid: np.ndarray, rule_text: str, steps: int,
                   f: int = 16, workers: int = 1, tile_w: int = 1, tile_h: int = 14,
                   inject_fault: bool = False, stats: bool = False):
        g = np.ascontiguousarray(grid, np.uint8)
        n = g.shape[0]
        out = np.empty_like(g)
        st = np.zeros(6, np.int64)
        self._check(self.lib.ref_run_engine(self.ENGINE[engine], n, f, _ptr(g, _u8p),
                                            rule_text.encode(), steps, workers, tile_w,
                                            tile_h, int(inject_fault), _ptr(out, _u8p),
                                            _ptr(st, _i64p)))
        if stats:
            keys = ("mma_count", "steps", "max_h", "max_r", "fragments_per_row", "accesses")
            return out, dict(zip(keys, (int(v) for v in st)))
        return out

    def run_cat_timed(self, grid: np.ndarray, rule_text: str, steps: int, workers: int = 1,
                      f: int = 16, want_output: bool = False):
        """run_engine(Cat) timed inside the library: (ms whole call incl. layout
        conversion, ms of simulate() alone[, output grid])."""
        g = np.ascontiguousarray(grid, np.uint8)
        out = np.empty_like(g) if want_output else None
        ms = (ctypes.c_double * 2)()
        self._check(self.lib.ref_run_cat_timed(g.shape[0], f, _ptr(g, _u8p), rule_text.encode(),
                                               steps, workers,
                                               _ptr(out, _u8p) if want_output else None, ms))
        return (ms[0], ms[1], out) if want_output else (ms[0], ms[1])

    def reductions(self, grid: np.ndarray, rule_text: str, f: int = 16):
        g = np.ascontiguousarray(grid, np.uint8)
        n = g.shape[0]
        p = n + 2 * f
        h = np.zeros((p, p), np.int32)
        red = np.zeros((p, p), np.int32)
        self._check(self.lib.ref_reductions(n, f, _ptr(g, _u8p), rule_text.encode(),
                                            _ptr(h, _i32p), _ptr(red, _i32p)))
        return h, red

    def semantic_steps(self, grid: np.ndarray, rule_ints, steps: int) -> np.ndarray:
        """tests/oracle.hpp torus_rule_steps: the reference's brute-force
        semantic oracle, any radius (no rule validation -- defines r > 16)."""
        g = np.ascontiguousarray(grid, np.uint8)
        out = np.empty_like(g)
        r8 = np.ascontiguousarray(rule_ints, np.int32)
        self._check(self.lib.ref_semantic_steps(g.shape[0], _ptr(g, _u8p), _ptr(r8, _i32p), steps,
                                                _ptr(out, _u8p)))
        return out

    def snapshot_write(self, grid: np.ndarray, path: str, f: int = 16, layout: int = 0) -> None:
        """catsim::snapshot_write of a row-major interior, as layout 0 / 1."""
        g = np.ascontiguousarray(grid, np.uint8)
        self._check(self.lib.ref_snapshot_write(g.shape[0], f, layout, _ptr(g, _u8p),
                                                path.encode()))

    def snapshot_read(self, path: str):
        """catsim::snapshot_read -> (interior, f, layout)."""
        n, f, lay = (np.zeros(1, np.int32) for _ in range(3))
        self._check(self.lib.ref_snapshot_read(path.encode(), _ptr(n, _i32p), _ptr(f, _i32p),
                                               _ptr(lay, _i32p), None, 0))
        out = np.zeros((int(n[0]), int(n[0])), np.uint8)
        self._check(self.lib.ref_snapshot_read(path.encode(), _ptr(n, _i32p), _ptr(f, _i32p),
                                               _ptr(lay, _i32p), _ptr(out, _u8p), out.size))
        return out, int(f[0]), int(lay[0])


def rule_text(rule) -> str:
    """format_ltl_rule (src/rule.cpp:89-97) for an 8-int rule vector."""
    r, c, m, s1, s2, b1, b2, kind = rule
    return f"R{r},C{c},M{m},S{s1}..{s2},B{b1}..{b2},N{'M' if kind == 0 else 'N'}"
