"""B200-native Larger-than-Life step (arXiv 2406.17284, CAT) -- drop-in for the
reference catsim CAT engine.  The compute lives in libltl_b200.so (sm_100a
CUDA + C-ABI, include/ltl_b200.h); this package is its Python binding."""
from .ltl import (  # noqa: F401
    DeviceTorus, LtlRule, LtlLogicError, LtlCudaError, find_preset, format_ltl_rule,
    load_library, ltl_presets, parse_ltl_rule, run_engine, von_neumann_probe_rule,
)
