"""B200-native Ozaki scheme II GEMM emulation (arXiv 2508.03984).

Drop-in for the reference C++ library's hot path (``crtgemm::gemm_emulated``):
the C ABI in include/ozaki2_b200.h, implemented by hand-written sm_100a CUDA
(paper_2508_03984_b200/csrc), mirrored here for Python callers.
"""
from .emulator import (  # noqa: F401
    ConfigError,
    Context,
    CudaError,
    EmuConfig,
    EmulationResult,
    InputError,
    Precision,
    ScaleMode,
    build_constants,
    default_context,
    dump_tables_csv,
    gemm_emulated,
    mod_inverse,
    select_moduli,
    to_fp32,
)
from .gen import gen_int_matrix, gen_matrix  # noqa: F401

__all__ = [
    "ConfigError", "Context", "CudaError", "EmuConfig", "EmulationResult", "InputError", "Precision", "ScaleMode",
    "build_constants", "default_context", "dump_tables_csv", "gemm_emulated", "mod_inverse", "select_moduli",
    "to_fp32", "gen_matrix", "gen_int_matrix",
]
