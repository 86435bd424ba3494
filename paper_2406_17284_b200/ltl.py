"""ctypes binding of libltl_b200.so (the C-ABI declared in include/ltl_b200.h).

This is the Python-side binding a maintainer would add to drive the B200
library from tests, benchmarks or notebooks (INTEGRATION.md shows the same for
cgo / JNI).  It mirrors the reference's engine front end
(proj/include/catsim/engines.hpp:13-25): ``run_engine`` takes a row-major grid,
runs `steps` generations and returns a row-major grid, and errors surface as
the reference's exception classes (ValueError ~ std::invalid_argument,
RuntimeError subclasses ~ std::logic_error) with the same message prefixes.

There is deliberately no CPU fallback: if the library is missing or no B200 is
visible, calls raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# LTL_LIB: load another build of the library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("LTL_LIB", os.path.join(HERE, "libltl_b200.so"))

OK, ERR_INVALID_ARGUMENT, ERR_LOGIC, ERR_RUNTIME, ERR_CUDA = range(5)
LAYOUT_ROW_MAJOR, LAYOUT_FRAGMENT = 0, 1
KIND_MOORE, KIND_VON_NEUMANN = 0, 1
FLAG_INJECT_FAULT, FLAG_WANT_STATS, FLAG_ENGINE_BASE, FLAG_ENGINE_PACK = 0x1, 0x2, 0x4, 0x10
# extension: the Cat engine with 17 <= r <= 32 (include/ltl_b200.h LTL_FLAG_WIDE_RADIUS);
# set automatically for rules with r > 16
FLAG_WIDE_RADIUS = 0x20
MAX_RADIUS, MAX_WIDE_RADIUS = 16, 32
FLAG_STENCIL = FLAG_ENGINE_BASE
# engine name -> ltl_run flag (catsim::EngineKind; proj/src/engines.cpp:9-15)
# the Cat engine on 4-bit device cells where the geometry allows (opt-in,
# include/ltl_b200.h LTL_FLAG_4BIT_CELLS; same bytes as "cat")
FLAG_4BIT_CELLS = 0x40
ENGINE_FLAGS = {"cat": 0, "base": FLAG_ENGINE_BASE, "pack": FLAG_ENGINE_PACK,
                "cat-4bit": FLAG_4BIT_CELLS}


class LtlLogicError(RuntimeError):
    """std::logic_error analogue (sequencing / internal consistency)."""


class LtlCudaError(RuntimeError):
    """Device failure (no reference analogue)."""


class LtlRuntimeError(RuntimeError):
    """std::runtime_error analogue."""


_EXC = {ERR_INVALID_ARGUMENT: ValueError, ERR_LOGIC: LtlLogicError,
        ERR_RUNTIME: LtlRuntimeError, ERR_CUDA: LtlCudaError}


class ltl_rule_c(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int32) for k in ("r", "c", "m", "s1", "s2", "b1", "b2", "kind")]


class ltl_stats_c(ctypes.Structure):
    _fields_ = [("mma_count", ctypes.c_int64), ("steps", ctypes.c_int64),
                ("max_h", ctypes.c_int32), ("max_r", ctypes.c_int32),
                ("fragments_per_row", ctypes.c_int32), ("reserved", ctypes.c_int32)]


# Every symbol include/ltl_b200.h declares (tests check the .so exports them all).
EXPORTS = (
    "ltl_create", "ltl_create_torus", "ltl_create_grid", "ltl_destroy", "ltl_last_error", "ltl_rows", "ltl_cols",
    "ltl_num_slabs", "ltl_kernel_launches", "ltl_time_launches", "ltl_transfer_bytes", "ltl_upload", "ltl_download",
    "ltl_upload_interior", "ltl_download_interior", "ltl_run", "ltl_run_async", "ltl_synchronize", "ltl_time",
    "ltl_run_interior", "ltl_create_part", "ltl_set_stream", "ltl_step_part", "ltl_fill_halo",
    "ltl_slab_buffer", "ltl_pack_edges", "ltl_unpack_halo", "ltl_ring_export",
    "ltl_ring_connect", "ltl_ring_fill", "ltl_ring_active", "ltl_ring_disconnect",
    "ltl_persistent_ok",
    "ltl_snapshot_write", "ltl_snapshot_read", "ltl_snapshot_probe", "ltl_snapshot_parse_header",
    "ltl_download_padded", "ltl_host_fill_halo",
    "ltl_fragment_pass",
    "ltl_init_random", "ltl_parse_rule", "ltl_parse_rule_ext", "ltl_format_rule",
    "ltl_preset_count", "ltl_preset", "ltl_von_neumann_probe_rule", "ltl_build_info",
)

_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the in-tree library (fails loudly when it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise FileNotFoundError(
            f"{path} not built; run `python -m paper_2406_17284_b200._build` (no CPU fallback)")
    lib = ctypes.CDLL(path)
    P = ctypes.POINTER
    vp, u8p = ctypes.c_void_p, P(ctypes.c_uint8)
    sig = {
        "ltl_create": ([P(vp), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P(ctypes.c_int32)],
                       ctypes.c_int),
        "ltl_create_torus": ([P(vp), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                              P(ctypes.c_int32)], ctypes.c_int),
        "ltl_create_grid": ([P(vp), ctypes.c_int32, ctypes.c_int32], ctypes.c_int),
        "ltl_destroy": ([vp], None),
        "ltl_last_error": ([vp], ctypes.c_char_p),
        "ltl_rows": ([vp], ctypes.c_int32),
        "ltl_cols": ([vp], ctypes.c_int32),
        "ltl_num_slabs": ([vp], ctypes.c_int32),
        "ltl_kernel_launches": ([vp], ctypes.c_int64),
        "ltl_time_launches": ([vp], ctypes.c_int64),
        "ltl_transfer_bytes": ([vp, ctypes.c_int32], ctypes.c_int64),
        "ltl_upload": ([vp, u8p, ctypes.c_int32], ctypes.c_int),
        "ltl_download": ([vp, u8p, ctypes.c_int32], ctypes.c_int),
        "ltl_download_padded": ([vp, u8p, ctypes.c_int32, ctypes.c_int32], ctypes.c_int),
        "ltl_host_fill_halo": ([u8p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32], ctypes.c_int),
        "ltl_snapshot_parse_header": ([ctypes.c_char_p, ctypes.c_int32, P(ctypes.c_int32),
                                       P(ctypes.c_int32), P(ctypes.c_int32)], ctypes.c_int),
        "ltl_upload_interior": ([vp, u8p], ctypes.c_int),
        "ltl_download_interior": ([vp, u8p], ctypes.c_int),
        "ltl_run": ([vp, P(ltl_rule_c), ctypes.c_int32, ctypes.c_uint32, P(ltl_stats_c)],
                    ctypes.c_int),
        "ltl_run_async": ([vp, P(ltl_rule_c), ctypes.c_int32, ctypes.c_uint32], ctypes.c_int),
        "ltl_synchronize": ([vp], ctypes.c_int),
        "ltl_time": ([vp, P(ltl_rule_c), ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32,
                      P(ctypes.c_double), P(ctypes.c_double)], ctypes.c_int),
        "ltl_run_interior": ([vp, u8p, u8p, P(ltl_rule_c), ctypes.c_int32, ctypes.c_uint32,
                              P(ltl_stats_c)], ctypes.c_int),
        "ltl_create_part": ([P(vp), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32],
                            ctypes.c_int),
        "ltl_set_stream": ([vp, ctypes.c_int32, vp], ctypes.c_int),
        "ltl_step_part": ([vp, P(ltl_rule_c), ctypes.c_uint32], ctypes.c_int),
        "ltl_fill_halo": ([vp], ctypes.c_int),
        "ltl_init_random": ([vp, ctypes.c_double, ctypes.c_uint64, ctypes.c_int32], ctypes.c_int),
        "ltl_slab_buffer": ([vp, ctypes.c_int32, ctypes.c_int32, P(vp), P(ctypes.c_int64),
                             P(ctypes.c_int32)], ctypes.c_int),
        "ltl_pack_edges": ([vp, vp, vp], ctypes.c_int),
        "ltl_ring_export": ([vp, vp], ctypes.c_int),
        "ltl_ring_connect": ([vp, vp, ctypes.c_int32, vp, ctypes.c_int32], ctypes.c_int),
        "ltl_ring_fill": ([vp], ctypes.c_int),
        "ltl_ring_active": ([vp], ctypes.c_int32),
        "ltl_ring_disconnect": ([vp], ctypes.c_int),
        "ltl_persistent_ok": ([vp, ctypes.c_uint32], ctypes.c_int32),
        "ltl_snapshot_write": ([vp, ctypes.c_char_p, ctypes.c_int32], ctypes.c_int),
        "ltl_snapshot_read": ([vp, ctypes.c_char_p, ctypes.POINTER(ctypes.c_int32)], ctypes.c_int),
        "ltl_snapshot_probe": ([ctypes.c_char_p, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)],
                               ctypes.c_int),
        "ltl_fragment_pass": ([ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, u8p,
                               P(ctypes.c_int32), P(ctypes.c_int32), P(ctypes.c_int32)],
                              ctypes.c_int),
        "ltl_unpack_halo": ([vp, vp, vp], ctypes.c_int),
        "ltl_parse_rule": ([ctypes.c_char_p, P(ltl_rule_c), ctypes.c_char_p, ctypes.c_int32],
                           ctypes.c_int),
        "ltl_parse_rule_ext": ([ctypes.c_char_p, ctypes.c_int32, P(ltl_rule_c), ctypes.c_char_p,
                                ctypes.c_int32], ctypes.c_int),
        "ltl_format_rule": ([P(ltl_rule_c), ctypes.c_char_p, ctypes.c_int32], ctypes.c_int32),
        "ltl_preset_count": ([], ctypes.c_int32),
        "ltl_preset": ([ctypes.c_int32, P(ctypes.c_char_p), P(ctypes.c_char_p),
                        P(ctypes.c_double)], ctypes.c_int),
        "ltl_von_neumann_probe_rule": ([ctypes.c_int32, P(ltl_rule_c)], None),
        "ltl_build_info": ([], ctypes.c_char_p),
    }
    for name, (args, res) in sig.items():
        if "LTL_LIB" in os.environ and not hasattr(lib, name):
            continue  # A/B against an older build: entry points it predates stay unbound
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


# ---------------------------------------------------------------- rules
@dataclass(frozen=True)
class LtlRule:
    """catsim::LtlRule (proj/include/catsim/rule.hpp:17-32)."""
    r: int = 1
    c: int = 2
    m: int = 0
    s1: int = 0
    s2: int = 0
    b1: int = 0
    b2: int = 0
    kind: int = KIND_MOORE

    def to_c(self) -> ltl_rule_c:
        return ltl_rule_c(self.r, self.c, self.m, self.s1, self.s2, self.b1, self.b2, self.kind)

    def ints(self):
        return [self.r, self.c, self.m, self.s1, self.s2, self.b1, self.b2, self.kind]

    @classmethod
    def from_c(cls, c: ltl_rule_c) -> "LtlRule":
        return cls(c.r, c.c, c.m, c.s1, c.s2, c.b1, c.b2, c.kind)

    def __str__(self) -> str:
        return format_ltl_rule(self)


def parse_ltl_rule(text: str, max_radius: int = MAX_RADIUS) -> LtlRule:
    """parse_ltl_rule (src/rule.cpp:61-87); max_radius up to 32 is the
    wide-radius extension (the reference stops at 16)."""
    lib = load_library()
    out = ltl_rule_c()
    err = ctypes.create_string_buffer(256)
    if lib.ltl_parse_rule_ext(text.encode(), max_radius, ctypes.byref(out), err, 256) != OK:
        raise ValueError(err.value.decode())
    return LtlRule.from_c(out)


def format_ltl_rule(rule: LtlRule) -> str:
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    c = rule.to_c()
    lib.ltl_format_rule(ctypes.byref(c), buf, 128)
    return buf.value.decode()


def ltl_presets():
    lib = load_library()
    out = []
    for i in range(lib.ltl_preset_count()):
        name, rule, dens = ctypes.c_char_p(), ctypes.c_char_p(), ctypes.c_double()
        lib.ltl_preset(i, ctypes.byref(name), ctypes.byref(rule), ctypes.byref(dens))
        out.append((name.value.decode(), rule.value.decode(), dens.value))
    return out


def find_preset(name: str):
    for p in ltl_presets():
        if p[0] == name:
            return p
    return None


def von_neumann_probe_rule(r: int) -> LtlRule:
    lib = load_library()
    out = ltl_rule_c()
    lib.ltl_von_neumann_probe_rule(r, ctypes.byref(out))
    return LtlRule.from_c(out)


def as_rule(rule) -> LtlRule:
    if isinstance(rule, LtlRule):
        return rule
    if isinstance(rule, str):
        return parse_ltl_rule(rule)
    return LtlRule(*[int(v) for v in rule])


# ---------------------------------------------------------------- device grid
def _u8(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))


class DeviceTorus:
    """A device-resident torus (one ltl_ctx): row slabs over one or more GPUs."""

    def __init__(self, n: int | None = None, f: int = 16, rows: int | None = None,
                 cols: int | None = None, slabs: int = 1, devices=None,
                 part_device: int | None = None, part_row0: int = 0):
        """n (square, fragment side f) or rows x cols (rectangular torus), split
        into `slabs` row slabs on `devices`.  part_device=d makes this context
        one rank's slab of a torus partitioned across processes: the rows above
        and below come from the caller's transport (see step_part)."""
        self.lib = load_library()
        self._ctx = ctypes.c_void_p()
        devs = None
        if devices is not None:
            devs = (ctypes.c_int32 * len(devices))(*devices)
        if part_device is not None:
            st = self.lib.ltl_create_part(ctypes.byref(self._ctx), rows, cols, part_row0, part_device)
        elif n is not None:
            st = self.lib.ltl_create(ctypes.byref(self._ctx), n, f, slabs, devs)
        else:
            st = self.lib.ltl_create_torus(ctypes.byref(self._ctx), rows, cols, slabs, devs)
        if st != OK:
            raise _EXC.get(st, RuntimeError)(self.lib.ltl_last_error(None).decode())
        self.rows = self.lib.ltl_rows(self._ctx)
        self.cols = self.lib.ltl_cols(self._ctx)
        self.f = f

    def _check(self, st: int):
        if st != OK:
            raise _EXC.get(st, RuntimeError)(self.lib.ltl_last_error(self._ctx).decode())

    def close(self):
        if self._ctx:
            self.lib.ltl_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def upload(self, interior: np.ndarray) -> None:
        a = np.ascontiguousarray(interior, np.uint8)
        if a.shape != (self.rows, self.cols):
            raise ValueError(f"geometry error: expected {(self.rows, self.cols)}, got {a.shape}")
        self._check(self.lib.ltl_upload_interior(self._ctx, _u8(a)))

    def download(self, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty((self.rows, self.cols), np.uint8)
        self._check(self.lib.ltl_download_interior(self._ctx, _u8(out)))
        return out

    def snapshot_write(self, path: str, layout: int = LAYOUT_ROW_MAJOR) -> None:
        """catsim::snapshot_write of the device grid, streamed (no host grid)."""
        self._check(self.lib.ltl_snapshot_write(self._ctx, os.fsencode(path), layout))

    def snapshot_read(self, path: str) -> int:
        """catsim::snapshot_read into the device grid; returns the declared layout."""
        lay = ctypes.c_int32(-1)
        self._check(self.lib.ltl_snapshot_read(self._ctx, os.fsencode(path), ctypes.byref(lay)))
        return lay.value

    def init_random(self, density: float, seed: int, fill_n: int = -1) -> None:
        """Device-side init_random (bit-identical to src/grid.cpp:61-73)."""
        self._check(self.lib.ltl_init_random(self._ctx, density, seed, fill_n))

    def upload_padded(self, padded: np.ndarray, layout: int = LAYOUT_ROW_MAJOR) -> None:
        a = np.ascontiguousarray(padded, np.uint8)
        self._check(self.lib.ltl_upload(self._ctx, _u8(a), layout))

    def download_padded(self, layout: int = LAYOUT_ROW_MAJOR) -> np.ndarray:
        p = self.rows + 2 * self.f
        out = np.empty(p * p, np.uint8)
        self._check(self.lib.ltl_download(self._ctx, _u8(out), layout))
        return out.reshape(p, p) if layout == LAYOUT_ROW_MAJOR else out

    @staticmethod
    def _flags(engine: str, inject_fault: bool = False, stencil: bool = False,
               rule: ltl_rule_c | None = None) -> int:
        """engine "cat" | "base" | "pack" (stencil=True: the round-1 spelling of
        "base"); a Cat rule with r > 16 adds FLAG_WIDE_RADIUS."""
        if stencil and engine == "cat":
            engine = "base"
        if engine not in ENGINE_FLAGS:
            raise ValueError(f"config error: unknown engine '{engine}' (cat, base, pack)")
        wide = engine in ("cat", "cat-4bit") and rule is not None and rule.r > MAX_RADIUS
        return (ENGINE_FLAGS[engine] | (FLAG_INJECT_FAULT if inject_fault else 0)
                | (FLAG_WIDE_RADIUS if wide else 0))

    def run(self, rule, steps: int, stencil: bool = False, inject_fault: bool = False,
            stats: bool = False, engine: str = "cat"):
        """`steps` generations.  stats=True returns the CatStats analogue (and
        runs the checked kernel variant that max-reduces H / R on the device)."""
        r = as_rule(rule).to_c()
        st = ltl_stats_c()
        flags = self._flags(engine, inject_fault, stencil, r) | (FLAG_WANT_STATS if stats else 0)
        self._check(self.lib.ltl_run(self._ctx, ctypes.byref(r), steps, flags,
                                     ctypes.byref(st) if stats else None))
        if not stats:
            return None
        return {k: getattr(st, k) for k, _ in ltl_stats_c._fields_ if k != "reserved"}

    def run_async(self, rule, steps: int, stencil: bool = False, engine: str = "cat") -> None:
        r = as_rule(rule).to_c()
        self._check(self.lib.ltl_run_async(self._ctx, ctypes.byref(r), steps,
                                           self._flags(engine, False, stencil, r)))

    def synchronize(self) -> None:
        self._check(self.lib.ltl_synchronize(self._ctx))

    def time(self, rule, steps: int, warmup: int = 3, stencil: bool = False,
             engine: str = "cat"):
        """(total_ms, kernel_ms) over `steps` generations, CUDA events, max over slabs."""
        r = as_rule(rule).to_c()
        tot, ker = ctypes.c_double(), ctypes.c_double()
        self._check(self.lib.ltl_time(self._ctx, ctypes.byref(r), steps, warmup,
                                      self._flags(engine, False, stencil, r), ctypes.byref(tot),
                                      ctypes.byref(ker)))
        return tot.value, ker.value

    def run_interior(self, interior: np.ndarray, rule, steps: int, out: np.ndarray | None = None,
                     stencil: bool = False, engine: str = "cat") -> np.ndarray:
        a = np.ascontiguousarray(interior, np.uint8)
        if out is None:
            out = np.empty_like(a)
        r = as_rule(rule).to_c()
        st = ltl_stats_c()
        self._check(self.lib.ltl_run_interior(self._ctx, _u8(a), _u8(out), ctypes.byref(r),
                                              steps, self._flags(engine, False, stencil, r),
                                              ctypes.byref(st)))
        return out

    def set_stream(self, stream_ptr: int, slab: int = 0) -> None:
        self._check(self.lib.ltl_set_stream(self._ctx, slab, ctypes.c_void_p(stream_ptr)))

    def step_part(self, rule, stencil: bool = False, engine: str = "cat") -> None:
        """Enqueue one generation + local column-halo refresh (async)."""
        r = as_rule(rule).to_c()
        self._check(self.lib.ltl_step_part(self._ctx, ctypes.byref(r),
                                           self._flags(engine, False, stencil, r)))

    def fill_halo(self) -> None:
        self._check(self.lib.ltl_fill_halo(self._ctx))

    def kernel_launches(self) -> int:
        """Kernels this context has launched so far (ltl_kernel_launches)."""
        return int(self.lib.ltl_kernel_launches(self._ctx))

    def time_launches(self) -> int:
        """Kernels launched inside the last time() call's timed loop."""
        return int(self.lib.ltl_time_launches(self._ctx))

    def transfer_bytes(self) -> tuple[int, int]:
        """(host -> device, device -> host) bytes moved so far (ltl_transfer_bytes)."""
        return (int(self.lib.ltl_transfer_bytes(self._ctx, 0)),
                int(self.lib.ltl_transfer_bytes(self._ctx, 1)))

    def slab_buffer(self, slab: int = 0, which: int = 0):
        """(device pointer, strip bytes, interior rows) of a generation buffer
        (column-strip layout, include/ltl_b200.h)."""
        ptr, strip_bytes, rows = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_int32()
        self._check(self.lib.ltl_slab_buffer(self._ctx, slab, which, ctypes.byref(ptr),
                                             ctypes.byref(strip_bytes), ctypes.byref(rows)))
        return ptr.value, strip_bytes.value, rows.value

    # ---- multi-process ring with the halo exchange fused into the step
    RING_HANDLE_BYTES = 4 * 64 + 32  # include/ltl_b200.h LTL_RING_HANDLE_BYTES

    def ring_export(self) -> bytes:
        """CUDA IPC handles of the slab's step counters and both generation buffers."""
        buf = ctypes.create_string_buffer(self.RING_HANDLE_BYTES)
        self._check(self.lib.ltl_ring_export(self._ctx, buf))
        return buf.raw

    def ring_connect(self, up: bytes, up_rows: int, down: bytes, down_rows: int) -> None:
        self._check(self.lib.ltl_ring_connect(self._ctx, up, up_rows, down, down_rows))

    def ring_fill(self) -> None:
        """Restart the ring's step counters (after every rank's upload; barriers around)."""
        self._check(self.lib.ltl_ring_fill(self._ctx))

    def ring_active(self) -> bool:
        return bool(self.lib.ltl_ring_active(self._ctx))

    def ring_disconnect(self) -> None:
        self._check(self.lib.ltl_ring_disconnect(self._ctx))

    def persistent_ok(self, engine: str = "cat") -> bool:
        """Would a multi-generation run use one persistent launch here?"""
        return bool(self.lib.ltl_persistent_ok(self._ctx, self._flags(engine)))

    def pack_edges(self, top_ptr: int, bot_ptr: int) -> None:
        """Enqueue: device buffers top/bot (16 x cols) <- first / last 16 interior rows."""
        self._check(self.lib.ltl_pack_edges(self._ctx, ctypes.c_void_p(top_ptr),
                                            ctypes.c_void_p(bot_ptr)))

    def unpack_halo(self, top_ptr: int, bot_ptr: int) -> None:
        """Enqueue: halo rows above / below <- device buffers (16 x cols each)."""
        self._check(self.lib.ltl_unpack_halo(self._ctx, ctypes.c_void_p(top_ptr),
                                             ctypes.c_void_p(bot_ptr)))


ENGINES = ("cat", "base", "pack", "cat-4bit")  # cat-4bit: the Cat engine on 4-bit device cells


def snapshot_probe(path: str):
    """Header of a CATSNAP v1 file -> (n, f, layout); the reader's header errors
    (LtlRuntimeError "snapshot format error: ...").  Host only."""
    lib = load_library()
    n, f, lay = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    st = lib.ltl_snapshot_probe(os.fsencode(path), ctypes.byref(n), ctypes.byref(f),
                                ctypes.byref(lay))
    if st != OK:
        raise _EXC.get(st, RuntimeError)(lib.ltl_last_error(None).decode())
    return n.value, f.value, lay.value


def run_engine(engine: str, initial: np.ndarray, rule, steps: int, f: int = 16,
               slabs: int = 1, inject_fault: bool = False, stats: bool = False):
    """Engine front end (proj/src/engines.cpp:26-46) over the device library.

    engine: "cat" -> tcgen05 banded-MMA path; "base" -> CUDA-core direct-sum
    stencil; "pack" -> CUDA-core packed sliding-window stencil (the GPU
    counterparts of the reference's BASE / PACK comparison engines; the
    reference's own CPU engines live only in the test oracle, never here).
    "stencil" is accepted as the round-1 name of "base".
    """
    if engine == "stencil":
        engine = "base"
    if engine not in ENGINES:
        raise ValueError(f"config error: unknown engine '{engine}' (cat, base, pack)")
    g = np.ascontiguousarray(initial, np.uint8)
    if g.ndim != 2 or g.shape[0] != g.shape[1]:
        raise ValueError("geometry error: expected a square grid")
    with DeviceTorus(n=g.shape[0], f=f, slabs=slabs) as t:
        t.upload(g)
        st = t.run(rule, steps, engine=engine, inject_fault=inject_fault, stats=stats)
        out = t.download()
    return (out, st) if stats else out
