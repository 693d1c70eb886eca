"""ctypes binding of the C ABI in include/ozaki2_b200.h.

The shared library is built in-tree (paper_2508_03984_b200/lib/) by
``__graft_entry__.build()`` / ``make -C paper_2508_03984_b200/csrc``. There is
no fallback: if the library is missing, or the process has no B200, every
entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# OZK_LIB_PATH: another build of the same library (A/B timing of two commits)
LIB_PATH = os.environ.get("OZK_LIB_PATH") or os.path.join(PKG_DIR, "lib", "libozaki2_b200.so")

OZK_OK, OZK_CONFIG_ERROR, OZK_INPUT_ERROR, OZK_CUDA_ERROR, OZK_DOMAIN_ERROR, OZK_INTERNAL_ERROR = range(6)
OZK_FP64, OZK_FP32 = 0, 1
OZK_FAST, OZK_ACCURATE = 0, 1
OZK_R64F, OZK_R32F = 0, 1
OZK_PRODUCTS_I32, OZK_PRODUCTS_U8 = 0, 1
OZK_FLAG_FAST_EXPONENT_FIX = 1
OZK_FLAG_TRANS_A = 2
OZK_FLAG_TRANS_B = 4
OZK_FLAG_ASYNC = 8
MAX_MODULI = 20
ENGINE_MAX_K = 1 << 17

# every symbol include/ozaki2_b200.h declares (checked by tests/test_abi.py)
EXPORTED_SYMBOLS = (
    "ozk_create", "ozk_destroy", "ozk_set_stream", "ozk_last_error", "ozk_version", "ozk_default_config",
    "ozk_select_moduli", "ozk_mod_inverse", "ozk_build_constants", "ozk_dump_tables_csv",
    "ozk_gemm", "ozk_gemm_host", "ozk_dgemm", "ozk_sgemm", "ozk_dgemm_ex", "ozk_gemm_strided_batched",
    "ozk_stage_scale", "ozk_plane_ld", "ozk_stage_residues", "ozk_stage_products", "ozk_stage_reconstruct",
    "ozk_kernel_launches", "ozk_profile", "ozk_profile_read", "ozk_k3_replays", "ozk_sync",
    "ozk_shard_begin", "ozk_shard_rowmax", "ozk_shard_end",
    "ozk_shard_stream_begin", "ozk_shard_stream_rows", "ozk_shard_stream_end",
    "ozk_int8_gemm", "ozk_int8_gemm_reference", "ozk_truncate_scale", "ozk_residues", "ozk_mod_u8_array", "ozk_accumulate", "ozk_crt_reduce",
    "ozk_unscale", "ozk_set_workspace_limit", "ozk_workspace_bytes", "ozk_last_plan",
    "ozk_release_workspace", "ozk_fast_floor",
)
PROFILE_SLOTS = ("scale", "residues", "products", "reconstruct", "total")


class ConfigError(ValueError):
    """crtgemm::ConfigError (errors.hpp:9)."""


class InputError(ValueError):
    """crtgemm::InputError (errors.hpp:14)."""


class CudaError(RuntimeError):
    """A CUDA failure inside the library (no CPU fallback exists)."""


class OzkConstants(C.Structure):
    _fields_ = [
        ("n_moduli", C.c_int32),
        ("precision", C.c_int32),
        ("moduli", C.c_int32 * MAX_MODULI),
        ("q", C.c_int64 * MAX_MODULI),
        ("beta", C.c_int32 * MAX_MODULI),
        ("P1", C.c_double),
        ("P2", C.c_double),
        ("P_inv", C.c_double),
        ("pp_fast", C.c_float),
        ("pp_accu", C.c_float),
        ("s1", C.c_double * MAX_MODULI),
        ("s2", C.c_double * MAX_MODULI),
        ("pinv64", C.c_double * MAX_MODULI),
        ("pinv32", C.c_float * MAX_MODULI),
        ("pinv_mulhi", C.c_int32 * MAX_MODULI),
        ("P_bits", C.c_int32),
        ("P_limbs", C.c_uint32 * 6),
    ]


class OzkConfig(C.Structure):
    _fields_ = [
        ("n_moduli", C.c_int32),
        ("mode", C.c_int32),
        ("precision", C.c_int32),
        ("a_type", C.c_int32),
        ("c_type", C.c_int32),
        ("flags", C.c_int32),
        ("block_k", C.c_int64),
        ("constants", C.POINTER(OzkConstants)),
    ]


_lib = None


def load() -> C.CDLL:
    """Load the product library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    i64, p, i32 = C.c_int64, C.c_void_p, C.c_int
    L.ozk_last_error.restype = C.c_char_p
    L.ozk_create.argtypes = [C.POINTER(p), i32]
    L.ozk_destroy.argtypes = [p]
    L.ozk_set_stream.argtypes = [p, p]
    L.ozk_default_config.restype = OzkConfig
    L.ozk_default_config.argtypes = [i32, i32, i32]
    L.ozk_select_moduli.argtypes = [i32, p]
    L.ozk_mod_inverse.restype = i64
    L.ozk_mod_inverse.argtypes = [i64, i64, C.POINTER(i32)]
    L.ozk_build_constants.argtypes = [i32, i32, C.POINTER(OzkConstants)]
    L.ozk_dump_tables_csv.argtypes = [C.POINTER(OzkConstants), C.c_char_p, i64]
    gemm_args = [p, C.POINTER(OzkConfig), i64, i64, i64, C.c_double, p, i64, p, i64, C.c_double, p, i64]
    L.ozk_gemm.argtypes = gemm_args
    L.ozk_gemm_host.argtypes = gemm_args
    L.ozk_dgemm.argtypes = [p, i32, i32, i64, i64, i64, C.c_double, p, i64, p, i64, C.c_double, p, i64]
    L.ozk_sgemm.argtypes = [p, i32, i32, i64, i64, i64, C.c_float, p, i64, p, i64, C.c_float, p, i64]
    L.ozk_dgemm_ex.argtypes = [p, i32, i32, C.c_char, C.c_char, i64, i64, i64, C.c_double, p, i64, p, i64,
                               C.c_double, p, i64]
    L.ozk_gemm_strided_batched.argtypes = [p, C.POINTER(OzkConfig), i64, i64, i64, C.c_double, p, i64, i64, p, i64, i64,
                                           C.c_double, p, i64, i64, i64]
    L.ozk_stage_scale.argtypes = [p, C.POINTER(OzkConfig), i64, i64, i64, p, i64, p, i64, p, p]
    L.ozk_set_workspace_limit.argtypes = [p, i64]
    L.ozk_workspace_bytes.restype = i64
    L.ozk_workspace_bytes.argtypes = [p]
    L.ozk_last_plan.argtypes = [p, p]
    L.ozk_release_workspace.argtypes = [p]
    L.ozk_fast_floor.argtypes = [C.c_float, C.c_double, i32]
    L.ozk_plane_ld.restype = i64
    L.ozk_plane_ld.argtypes = [i64]
    L.ozk_stage_residues.argtypes = [p, C.POINTER(OzkConfig), i64, i64, i64, p, i64, p, i64, p, p, p, p]
    L.ozk_stage_products.argtypes = [p, C.POINTER(OzkConfig), i64, i64, i64, p, p, i32, p, i64]
    L.ozk_stage_reconstruct.argtypes = [p, C.POINTER(OzkConfig), i64, i64, p, i64, p, p, C.c_double, C.c_double,
                                        p, i64]
    L.ozk_kernel_launches.restype = i64
    L.ozk_kernel_launches.argtypes = [p]
    L.ozk_profile.argtypes = [p, i32]
    L.ozk_sync.argtypes = [p]
    L.ozk_shard_begin.argtypes = [p, C.POINTER(OzkConfig), i64, i64, i64, p, i64, p, i64]
    L.ozk_shard_rowmax.restype = p
    L.ozk_shard_rowmax.argtypes = [p]
    L.ozk_shard_end.argtypes = [p, C.c_double, C.c_double, p, i64]
    L.ozk_shard_stream_begin.argtypes = [p, C.POINTER(OzkConfig), i64, i64, i64, p, i64, C.c_double, C.c_double,
                                         p, i64]
    L.ozk_shard_stream_rows.argtypes = [p, i64, i64, p, i64]
    L.ozk_shard_stream_end.argtypes = [p]
    L.ozk_int8_gemm.argtypes = [p, i64, i64, i64, p, i64, p, i64, p, i64]
    L.ozk_int8_gemm_reference.argtypes = [p, i64, i64, i64, p, i64, p, i64, p, i64]
    L.ozk_truncate_scale.argtypes = [p, i32, i64, i64, p, i64, p, i32, p, i64]
    L.ozk_residues.argtypes = [p, C.POINTER(OzkConfig), i64, i64, p, i64, p, i64]
    L.ozk_mod_u8_array.argtypes = [p, i64, p, C.c_int32, C.c_int32, p]
    L.ozk_accumulate.argtypes = [p, C.POINTER(OzkConfig), i64, p, p, p]
    L.ozk_crt_reduce.argtypes = [p, C.POINTER(OzkConfig), i64, p, p, p]
    L.ozk_unscale.argtypes = [p, i64, i64, p, i64, p, p, p, i64]
    L.ozk_profile_read.argtypes = [p, p, p, i32]
    L.ozk_k3_replays.argtypes = [p, p, i32]
    _lib = L
    return L


def check(status: int) -> None:
    if status == OZK_OK:
        return
    msg = load().ozk_last_error().decode(errors="replace")
    if status == OZK_CONFIG_ERROR:
        raise ConfigError(msg)
    if status == OZK_INPUT_ERROR:
        raise InputError(msg)
    if status == OZK_DOMAIN_ERROR:
        raise ArithmeticError(msg)
    raise CudaError(f"status {status}: {msg}")
