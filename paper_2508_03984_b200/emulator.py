"""Python mirror of the reference C++ API (crtgemm, emulator.hpp:12-35).

Same names, argument meaning and error behaviour as the reference:
``gemm_emulated(a, b, cfg)`` takes column-major host matrices (numpy arrays;
Fortran order is used as-is, anything else is copied) and returns an
``EmulationResult`` whose ``c`` is FP64 for both precisions (emulator.hpp:20-22).
Bad configurations raise ``ConfigError``, bad inputs ``InputError``
(errors.hpp:8-16). The work runs on the B200 through the C ABI; the Python
layer only marshals buffers.

``Context`` exposes the device-pointer API (torch CUDA tensors, column-major:
an m x k matrix is a tensor of shape (m, k) with stride (1, ld)) and the
stage-level exports used by the parity tests.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import threading

import numpy as np

from . import _lib
from ._lib import ConfigError, CudaError, InputError  # noqa: F401  (re-exported)


class Precision(enum.IntEnum):
    Fp64 = _lib.OZK_FP64
    Fp32 = _lib.OZK_FP32


class ScaleMode(enum.IntEnum):
    Fast = _lib.OZK_FAST
    Accurate = _lib.OZK_ACCURATE


kEngineMaxK = _lib.ENGINE_MAX_K


@dataclasses.dataclass
class EmuConfig:
    """emulator.hpp:12-18."""
    n_moduli: int = 15
    mode: ScaleMode = ScaleMode.Fast
    precision: Precision = Precision.Fp64
    block_k: int = kEngineMaxK
    threads: int = 1
    # extension (not in the reference): subtract the max exponent in fast-mode
    # scaling, the term scaling.cpp:50-56 omits. Off = reference bits.
    fast_exponent_fix: bool = False
    # extension: stream-ordered device calls (OZK_FLAG_ASYNC) — no host sync per
    # call, CUDA-graph capturable; the non-finite check is collected by
    # Context.synchronize(). Host-buffer calls ignore it.
    stream_ordered: bool = False


@dataclasses.dataclass
class EmulationResult:
    """reconstruct.hpp:21-26."""
    c: np.ndarray
    n_moduli: int
    mode: ScaleMode
    precision: Precision


def build_constants(n_moduli: int, precision: Precision = Precision.Fp64) -> _lib.OzkConstants:
    """crt_tables.hpp:71 (ConfigError for N outside the precision's range)."""
    L = _lib.load()
    c = _lib.OzkConstants()
    _lib.check(L.ozk_build_constants(int(n_moduli), int(precision), C.byref(c)))
    return c


def select_moduli(n_moduli: int) -> list:
    L = _lib.load()
    buf = (C.c_int32 * _lib.MAX_MODULI)()
    _lib.check(L.ozk_select_moduli(int(n_moduli), buf))
    return list(buf[:n_moduli])


def mod_inverse(a: int, m: int) -> int:
    L = _lib.load()
    st = C.c_int(0)
    r = L.ozk_mod_inverse(int(a), int(m), C.byref(st))
    _lib.check(st.value)
    return int(r)


def dump_tables_csv(c: _lib.OzkConstants) -> str:
    L = _lib.load()
    buf = C.create_string_buffer(8192)
    _lib.check(L.ozk_dump_tables_csv(C.byref(c), buf, 8192))
    return buf.value.decode()


def _config(cfg: EmuConfig, a_type: int, c_type: int, constants=None, trans_a: bool = False,
            trans_b: bool = False) -> _lib.OzkConfig:
    c = _lib.OzkConfig()
    c.n_moduli = int(cfg.n_moduli)
    c.mode = int(cfg.mode)
    c.precision = int(cfg.precision)
    c.a_type = a_type
    c.c_type = c_type
    c.block_k = int(cfg.block_k)
    c.flags = _lib.OZK_FLAG_FAST_EXPONENT_FIX if getattr(cfg, "fast_exponent_fix", False) else 0
    c.flags |= (_lib.OZK_FLAG_TRANS_A if trans_a else 0) | (_lib.OZK_FLAG_TRANS_B if trans_b else 0)
    c.flags |= _lib.OZK_FLAG_ASYNC if getattr(cfg, "stream_ordered", False) else 0
    c.constants = C.pointer(constants) if constants is not None else None
    return c


class Context:
    """An ozk_handle bound to one device (and optionally a CUDA stream)."""

    def __init__(self, device: int = 0):
        L = _lib.load()
        h = C.c_void_p()
        _lib.check(L.ozk_create(C.byref(h), int(device)))
        self.handle = h
        self.device = device
        self._lib = L

    def close(self) -> None:
        if self.handle:
            self._lib.ozk_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_workspace_limit(self, nbytes: int) -> None:
        """device workspace cap in bytes (0: automatic); larger problems run in panels"""
        _lib.check(self._lib.ozk_set_workspace_limit(self.handle, int(nbytes)))

    def release_workspace(self) -> None:
        """free the handle's device workspace (planes, U, staging)"""
        _lib.check(self._lib.ozk_release_workspace(self.handle))

    @property
    def workspace_bytes(self) -> int:
        return int(self._lib.ozk_workspace_bytes(self.handle))

    @property
    def last_plan(self) -> dict:
        """the panel plan of the last gemm: row panel height, column panel width, panels, extra residue passes"""
        out = (C.c_int64 * 4)()
        _lib.check(self._lib.ozk_last_plan(self.handle, out))
        return {"rows": out[0], "cols": out[1], "panels": out[2], "extra_passes": out[3]}

    def set_stream(self, stream_ptr: int) -> None:
        _lib.check(self._lib.ozk_set_stream(self.handle, C.c_void_p(stream_ptr)))

    @property
    def kernel_launches(self) -> int:
        return int(self._lib.ozk_kernel_launches(self.handle))

    def profile(self, enable: bool = True) -> None:
        _lib.check(self._lib.ozk_profile(self.handle, int(enable)))

    def profile_read(self, reset: bool = True) -> dict:
        """{stage: (total_ms, calls)} accumulated since the last reset"""
        ms = (C.c_double * len(_lib.PROFILE_SLOTS))()
        calls = (C.c_int64 * len(_lib.PROFILE_SLOTS))()
        _lib.check(self._lib.ozk_profile_read(self.handle, ms, calls, int(reset)))
        return {name: (ms[i], calls[i]) for i, name in enumerate(_lib.PROFILE_SLOTS)}

    def k3_replays(self, reset: bool = True) -> int:
        """elements whose C2 the tensor-core K3 replayed sequentially on this
        context's device since counting began there (the first call starts it)"""
        n = C.c_ulonglong(0)
        _lib.check(self._lib.ozk_k3_replays(self.handle, C.byref(n), int(reset)))
        return int(n.value)

    # ---- host (reference-facing) GEMM ----------------------------------------------
    def gemm_host(self, a: np.ndarray, b: np.ndarray, cfg: EmuConfig, alpha: float = 1.0, beta: float = 0.0,
                  c: np.ndarray | None = None, c_dtype=np.float64, constants=None, trans_a: bool = False,
                  trans_b: bool = False) -> np.ndarray:
        """C = alpha op(a) op(b) + beta c with op(x) = x.T when trans_x (a/b are
        passed as stored, e.g. a is k x m for trans_a; nothing is transposed)."""
        _validate_threads(a.T if trans_a else a, b.T if trans_b else b, cfg)
        dt = np.float32 if a.dtype == np.float32 else np.float64
        # column-major views with a leading dimension > rows (e.g. big[:m, :])
        # pass through as (pointer, ld), like a BLAS submatrix
        a, lda = _host_colmajor(a, dt)
        b, ldb = _host_colmajor(b, dt)
        m, k = (a.shape[1], a.shape[0]) if trans_a else a.shape
        n = b.shape[0] if trans_b else b.shape[1]
        out = np.zeros((m, n), dtype=c_dtype, order="F") if c is None else c
        ldc = _host_ld(out)
        if ldc is None or out.shape != (m, n):
            raise InputError("c must be an m x n column-major array (Fortran order, or a column-major view)")
        conf = _config(cfg, _lib.OZK_R32F if dt == np.float32 else _lib.OZK_R64F,
                       _lib.OZK_R32F if out.dtype == np.float32 else _lib.OZK_R64F, constants, trans_a, trans_b)
        _lib.check(self._lib.ozk_gemm_host(self.handle, C.byref(conf), m, n, k, float(alpha), a.ctypes.data,
                                           lda, b.ctypes.data, ldb, float(beta), out.ctypes.data, ldc))
        return out

    def synchronize(self) -> None:
        """wait for the handle's stream; raises InputError if a stream-ordered call
        since the last synchronize saw a non-finite input (ozk_sync)"""
        _lib.check(self._lib.ozk_sync(self.handle))

    # ---- device GEMM (torch CUDA tensors, column-major) ------------------------------
    def gemm(self, A, B, cfg: EmuConfig, C_out, alpha: float = 1.0, beta: float = 0.0, constants=None,
             trans_a: bool = False, trans_b: bool = False) -> None:
        """C_out = alpha op(A) op(B) + beta C_out; A, B as stored (column-major),
        op(X) = X^T when trans_x (BLAS 'T')."""
        m, k = (A.shape[1], A.shape[0]) if trans_a else A.shape
        n = B.shape[0] if trans_b else B.shape[1]
        lda, ldb, ldc = _colmajor_ld(A), _colmajor_ld(B), _colmajor_ld(C_out)
        conf = _config(cfg, _dtype_code(A), _dtype_code(C_out), constants, trans_a, trans_b)
        _lib.check(self._lib.ozk_gemm(self.handle, C.byref(conf), m, n, k, float(alpha), A.data_ptr(), lda,
                                      B.data_ptr(), ldb, float(beta), C_out.data_ptr(), ldc))

    def gemm_strided_batched(self, A, B, cfg: EmuConfig, C_out, alpha: float = 1.0, beta: float = 0.0,
                             trans_a: bool = False, trans_b: bool = False) -> None:
        """batched gemm over (batch, rows, cols) tensors whose slices are column-major
        (stride (s, 1, ld)), cublasGemmStridedBatched-style."""
        batch = A.shape[0]
        if B.shape[0] != batch or C_out.shape[0] != batch:
            raise InputError("batch sizes disagree")
        m, k = (A.shape[2], A.shape[1]) if trans_a else A.shape[1:]
        n = B.shape[1] if trans_b else B.shape[2]
        lda, ldb, ldc = _colmajor_ld(A[0]), _colmajor_ld(B[0]), _colmajor_ld(C_out[0])
        conf = _config(cfg, _dtype_code(A), _dtype_code(C_out), None, trans_a, trans_b)
        _lib.check(self._lib.ozk_gemm_strided_batched(
            self.handle, C.byref(conf), m, n, k, float(alpha), A.data_ptr(), lda, A.stride(0), B.data_ptr(), ldb,
            B.stride(0), float(beta), C_out.data_ptr(), ldc, C_out.stride(0), batch))

    # ---- column shard (multi-GPU, see distributed.py) -------------------------------
    def shard_begin(self, A, B, cfg: EmuConfig) -> None:
        m, k = A.shape
        n = B.shape[1]
        self._shard_m = m
        self._shard_conf = _config(cfg, _dtype_code(A), _lib.OZK_R64F)
        _lib.check(self._lib.ozk_shard_begin(self.handle, C.byref(self._shard_conf), m, n, k, A.data_ptr(),
                                             _colmajor_ld(A), B.data_ptr(), _colmajor_ld(B)))

    def shard_rowmax(self):
        """the m int32 partial row maxima on the device, as a torch tensor (no copy)"""
        import torch

        ptr = self._lib.ozk_shard_rowmax(self.handle)
        if not ptr:
            raise InputError("no open shard")

        class _Dev:
            __cuda_array_interface__ = {"shape": (self._shard_m,), "typestr": "<i4", "data": (ptr, False),
                                        "version": 3}

        return torch.as_tensor(_Dev(), device=f"cuda:{self.device}")

    def shard_end(self, C_out, alpha: float = 1.0, beta: float = 0.0) -> None:
        if C_out.dtype.itemsize == 4:
            raise InputError("shard output must be FP64 (set c_type through Context.gemm for FP32)")
        _lib.check(self._lib.ozk_shard_end(self.handle, float(alpha), float(beta), C_out.data_ptr(),
                                           _colmajor_ld(C_out)))

    # ---- row-streamed column shard (fast mode; A arrives in row blocks) --------------
    def shard_stream_begin(self, m: int, k: int, B, cfg: EmuConfig, C_out, alpha: float = 1.0,
                           beta: float = 0.0) -> None:
        """B's columns (this shard) are scaled and reduced now; C_out (m x n, FP64
        or FP32) receives alpha A B + beta C_out as the row blocks of A arrive."""
        n = B.shape[1]
        self._stream_conf = _config(cfg, _dtype_code(B), _dtype_code(C_out))
        _lib.check(self._lib.ozk_shard_stream_begin(self.handle, C.byref(self._stream_conf), m, n, k, B.data_ptr(),
                                                    _colmajor_ld(B), float(alpha), float(beta), C_out.data_ptr(),
                                                    _colmajor_ld(C_out)))

    def shard_stream_rows(self, r0: int, A_rows) -> None:
        """rows [r0, r0 + A_rows.shape[0]) of A as a column-major device block"""
        _lib.check(self._lib.ozk_shard_stream_rows(self.handle, r0, A_rows.shape[0], A_rows.data_ptr(),
                                                   _colmajor_ld(A_rows)))

    def shard_stream_end(self) -> None:
        _lib.check(self._lib.ozk_shard_stream_end(self.handle))

    # ---- stage exports (device tensors) --------------------------------------------
    def stage_scale(self, A, B, cfg: EmuConfig, mu_exp, nu_exp) -> None:
        m, k = A.shape
        n = B.shape[1]
        conf = _config(cfg, _dtype_code(A), _lib.OZK_R64F)
        _lib.check(self._lib.ozk_stage_scale(self.handle, C.byref(conf), m, n, k, A.data_ptr(), _colmajor_ld(A),
                                             B.data_ptr(), _colmajor_ld(B), mu_exp.data_ptr(), nu_exp.data_ptr()))

    def plane_ld(self, k: int) -> int:
        return int(self._lib.ozk_plane_ld(int(k)))

    def stage_residues(self, A, B, cfg: EmuConfig, mu_exp, nu_exp, a_planes, b_planes) -> None:
        m, k = A.shape
        n = B.shape[1]
        conf = _config(cfg, _dtype_code(A), _lib.OZK_R64F)
        _lib.check(self._lib.ozk_stage_residues(self.handle, C.byref(conf), m, n, k, A.data_ptr(), _colmajor_ld(A),
                                                B.data_ptr(), _colmajor_ld(B), mu_exp.data_ptr(), nu_exp.data_ptr(),
                                                a_planes.data_ptr(), b_planes.data_ptr()))

    def stage_products(self, cfg: EmuConfig, m: int, n: int, k: int, a_planes, b_planes, kind: int, out,
                       ldo: int) -> None:
        conf = _config(cfg, _lib.OZK_R64F, _lib.OZK_R64F)
        _lib.check(self._lib.ozk_stage_products(self.handle, C.byref(conf), m, n, k, a_planes.data_ptr(),
                                                b_planes.data_ptr(), int(kind), out.data_ptr(), int(ldo)))

    def stage_reconstruct(self, cfg: EmuConfig, m: int, n: int, U, ldu: int, mu_exp, nu_exp, C_out,
                          alpha: float = 1.0, beta: float = 0.0) -> None:
        conf = _config(cfg, _lib.OZK_R64F, _dtype_code(C_out))
        _lib.check(self._lib.ozk_stage_reconstruct(self.handle, C.byref(conf), m, n, U.data_ptr(), int(ldu),
                                                   mu_exp.data_ptr(), nu_exp.data_ptr(), float(alpha), float(beta),
                                                   C_out.data_ptr(), _colmajor_ld(C_out)))


def _host_ld(x: np.ndarray):
    """leading dimension of a column-major host matrix or view, else None"""
    if x.ndim != 2:
        return None
    it = x.itemsize
    if x.shape[1] <= 1 and (x.shape[0] <= 1 or x.strides[0] == it):
        return max(x.shape[0], 1)
    if x.strides[0] != it and x.shape[0] > 1:
        return None
    if x.strides[1] % it or x.strides[1] < it * x.shape[0]:
        return None
    return max(x.strides[1] // it, x.shape[0], 1)


def _host_colmajor(x: np.ndarray, dt):
    """(array, ld): x itself when it is a column-major matrix/view of dtype dt, else a Fortran copy"""
    ld = _host_ld(x) if x.dtype == dt else None
    if ld is None:
        x = np.asfortranarray(x, dtype=dt)
        ld = max(x.shape[0], 1)
    return x, ld


def _dtype_code(t) -> int:
    import torch

    if t.dtype == torch.float64:
        return _lib.OZK_R64F
    if t.dtype == torch.float32:
        return _lib.OZK_R32F
    raise InputError(f"unsupported dtype {t.dtype}")


def _colmajor_ld(t) -> int:
    if t.dim() != 2 or t.stride(0) != 1:
        raise InputError("expected a column-major matrix (tensor of shape (rows, cols) with stride (1, ld))")
    return max(int(t.stride(1)), int(t.shape[0]), 1)


def _validate_threads(a, b, cfg: EmuConfig) -> None:
    # the host-visible part of validate_inputs (emulator.cpp:14-18), same order
    if a.shape[1] != b.shape[0]:
        raise InputError("gemm_emulated: inner dimensions disagree")
    if min(a.shape[0], a.shape[1], b.shape[1]) < 1:
        raise InputError("gemm_emulated: empty dimension")
    if cfg.block_k < 1 or cfg.block_k > kEngineMaxK:
        raise ConfigError("gemm_emulated: block_k must be in [1, 2^17]")
    if cfg.threads < 1:
        raise ConfigError("gemm_emulated: threads must be >= 1")


_default_ctx = None
_ctx_lock = threading.Lock()


def default_context() -> Context:
    global _default_ctx
    with _ctx_lock:
        if _default_ctx is None:
            _default_ctx = Context(0)
        return _default_ctx


def gemm_emulated(a: np.ndarray, b: np.ndarray, cfg: EmuConfig, constants=None) -> EmulationResult:
    """emulator.hpp:23-32: C ~= A*B via Ozaki scheme II on the B200 tensor cores.

    FP32 inputs require ``cfg.precision == Fp32`` (emulator.cpp:97-98); FP64
    inputs with an Fp32 config are rounded to FP32 first (emulator.cpp:84-91).
    """
    if constants is None:
        constants = build_constants(cfg.n_moduli, cfg.precision)
    if a.dtype == np.float32 and cfg.precision != Precision.Fp32:
        raise ConfigError("gemm_emulated: FP32 inputs require cfg.precision == Fp32")
    _validate_threads(a, b, cfg)
    c = default_context().gemm_host(a, b, cfg, constants=constants)
    return EmulationResult(c=c, n_moduli=int(constants.n_moduli), mode=cfg.mode,
                           precision=Precision(int(constants.precision)))


def to_fp32(m: np.ndarray) -> np.ndarray:
    """emulator.cpp:110-115."""
    return np.asfortranarray(m, dtype=np.float32)
