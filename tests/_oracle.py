"""ctypes bindings for the two CPU checkers under oracle/ (TEST INFRASTRUCTURE).

* ``Oracle``  -> oracle/_lib/libozk_oracle.so, the plain-C restatement
  (oracle/ozk_oracle.c).
* ``RefLib``  -> oracle/_ref/libcrtgemm_ref.so, the unmodified reference
  sources compiled through the GMP header shim (oracle/Makefile). Present only
  where it was built (here, and on the GPU box through the gpurun snapshot).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use these.
All matrices are numpy arrays in Fortran (column-major) order, matching the
reference's Matrix<T> (matrix.hpp:9-32).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "_lib", "libozk_oracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libcrtgemm_ref.so")

_i64 = C.c_int64
_p = C.c_void_p


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _f(a, dtype):
    return np.asfortranarray(a, dtype=dtype)


class Constants(C.Structure):
    _fields_ = [
        ("n_moduli", C.c_int),
        ("precision", C.c_int),
        ("moduli", C.c_int * 20),
        ("q", C.c_long * 20),
        ("beta", C.c_int * 20),
        ("P1", C.c_double),
        ("P2", C.c_double),
        ("P_inv", C.c_double),
        ("pp_fast", C.c_float),
        ("pp_accu", C.c_float),
        ("s1", C.c_double * 20),
        ("s2", C.c_double * 20),
        ("pinv64", C.c_double * 20),
        ("pinv32", C.c_float * 20),
        ("pinv_mulhi", C.c_int32 * 20),
        ("P_bits", C.c_int),
    ]

    def as_dict(self) -> dict:
        n = self.n_moduli
        return {
            "moduli": list(self.moduli[:n]),
            "q": list(self.q[:n]),
            "beta": list(self.beta[:n]),
            "P1": self.P1,
            "P2": self.P2,
            "P_inv": self.P_inv,
            "pp_fast": np.float32(self.pp_fast),
            "pp_accu": np.float32(self.pp_accu),
            "s1": list(self.s1[:n]),
            "s2": list(self.s2[:n]),
            "pinv64": list(self.pinv64[:n]),
            "pinv32": [np.float32(x) for x in self.pinv32[:n]],
            "pinv_mulhi": list(self.pinv_mulhi[:n]),
            "P_bits": self.P_bits,
        }


def build_oracle() -> None:
    """(Re)build the plain-C oracle if missing (gcc is on both hosts)."""
    if not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-s", "-C", ORACLE_DIR, "oracle"], check=True)


class Oracle:
    """The plain-C restatement (oracle/ozk_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        build_oracle()
        L = self.lib = C.CDLL(path)
        L.ozo_build_constants.argtypes = [C.c_int, C.c_int, C.POINTER(Constants)]
        L.ozo_select_moduli.argtypes = [C.c_int, _p]
        L.ozo_mod_inverse.restype = C.c_long
        L.ozo_mod_inverse.argtypes = [C.c_long, C.c_long, C.POINTER(C.c_int)]
        for nm in ("ozo_scale_f64", "ozo_scale_f32"):
            getattr(L, nm).argtypes = [_p, _p, _i64, _i64, _i64, C.POINTER(Constants), C.c_int, _i64, _p, _p]
        for nm in ("ozo_truncate_f64", "ozo_truncate_f32"):
            getattr(L, nm).argtypes = [_p, _i64, _i64, _p, C.c_int, _p]
        L.ozo_rmod_fast_f64.restype = C.c_int8
        L.ozo_rmod_fast_f64.argtypes = [C.c_double, C.c_int, C.c_double, C.c_float, C.c_int]
        L.ozo_rmod_fast_f32.restype = C.c_int8
        L.ozo_rmod_fast_f32.argtypes = [C.c_float, C.c_int, C.c_float, C.c_int]
        for nm in ("ozo_residues_f64", "ozo_residues_f32"):
            getattr(L, nm).argtypes = [_p, _i64, C.POINTER(Constants), _p]
        L.ozo_int8_gemm.argtypes = [_p, _p, _i64, _i64, _i64, _p]
        L.ozo_mod_u8.restype = C.c_uint8
        L.ozo_mod_u8.argtypes = [C.c_int32, C.c_int32, C.c_int32]
        L.ozo_accumulate.argtypes = [_p, _i64, C.POINTER(Constants), _p, _p]
        L.ozo_crt_reduce_element.restype = C.c_double
        L.ozo_crt_reduce_element.argtypes = [C.c_double, C.c_double, C.POINTER(Constants)]
        L.ozo_unscale.argtypes = [_p, _i64, _i64, _p, _p, _p]
        for nm in ("ozo_gemm_f64", "ozo_gemm_f32", "ozo_products_u8_f64"):
            getattr(L, nm).argtypes = [_p, _p, _i64, _i64, _i64, C.c_int, C.c_int, _i64, _p]
        L.ozo_gemm_f64_consts.argtypes = [_p, _p, _i64, _i64, _i64, C.POINTER(Constants), C.c_int, _i64, _p]
        L.ozo_gemm_f64_scaled.argtypes = [_p, _p, _i64, _i64, _i64, C.POINTER(Constants), _p, _p, _i64, _p]
        L.ozo_gemm_f32_scaled.argtypes = [_p, _p, _i64, _i64, _i64, C.POINTER(Constants), _p, _p, _i64, _p]
        L.ozo_accurate_exponent.argtypes = [C.c_int64, C.c_int, C.POINTER(Constants)]

    # -- constants -----------------------------------------------------------------
    def constants(self, n: int, prec: int = 0) -> Constants:
        c = Constants()
        st = self.lib.ozo_build_constants(n, prec, C.byref(c))
        if st:
            raise ValueError(f"ConfigError (status {st})")
        return c

    def select_moduli(self, n: int) -> list:
        out = np.zeros(20, dtype=np.int32)
        if self.lib.ozo_select_moduli(n, _ptr(out)):
            raise ValueError("ConfigError")
        return out[:n].tolist()

    def mod_inverse(self, a: int, m: int) -> int:
        st = C.c_int(0)
        r = self.lib.ozo_mod_inverse(a, m, C.byref(st))
        if st.value:
            raise ArithmeticError("domain_error")
        return r

    # -- stages ----------------------------------------------------------------------
    def scale(self, a, b, n_moduli, mode, prec=0, block_k=1 << 17):
        dt = np.float64 if prec == 0 else np.float32
        a, b = _f(a, dt), _f(b, dt)
        m, k = a.shape
        n = b.shape[1]
        c = self.constants(n_moduli, prec)
        mu = np.zeros(m, np.int32)
        nu = np.zeros(n, np.int32)
        fn = self.lib.ozo_scale_f64 if prec == 0 else self.lib.ozo_scale_f32
        fn(_ptr(a), _ptr(b), m, n, k, C.byref(c), mode, block_k, _ptr(mu), _ptr(nu))
        return mu, nu

    def truncate(self, x, scale_exp, side, prec=0):
        dt = np.float64 if prec == 0 else np.float32
        x = _f(x, dt)
        se = np.ascontiguousarray(scale_exp, np.int32)
        out = np.zeros_like(x, order="F")
        fn = self.lib.ozo_truncate_f64 if prec == 0 else self.lib.ozo_truncate_f32
        fn(_ptr(x), x.shape[0], x.shape[1], _ptr(se), side, _ptr(out))
        return out

    def residues(self, xp, n_moduli, prec=0):
        """N column-major planes of xp (shape (N, rows, cols), Fortran per plane)."""
        dt = np.float64 if prec == 0 else np.float32
        xp = _f(xp, dt)
        c = self.constants(n_moduli, prec)
        planes = np.zeros((n_moduli, xp.size), np.int8)
        fn = self.lib.ozo_residues_f64 if prec == 0 else self.lib.ozo_residues_f32
        fn(_ptr(xp), xp.size, C.byref(c), _ptr(planes))
        return planes.reshape(n_moduli, xp.shape[1], xp.shape[0]).transpose(0, 2, 1)

    def int8_gemm(self, a, b):
        a, b = _f(a, np.int8), _f(b, np.int8)
        m, k = a.shape
        n = b.shape[1]
        c = np.zeros((m, n), np.int32, order="F")
        self.lib.ozo_int8_gemm(_ptr(a), _ptr(b), m, n, k, _ptr(c))
        return c

    def mod_u8(self, x: int, p: int, pinv: int) -> int:
        return self.lib.ozo_mod_u8(x, p, pinv)

    def accumulate(self, u, n_moduli, prec=0):
        """u: (N, rows, cols) uint8 -> (c1, c2) column-major."""
        c = self.constants(n_moduli, prec)
        N, r, cc = u.shape
        flat = np.ascontiguousarray(np.stack([np.asfortranarray(u[i]).ravel(order="F") for i in range(N)]))
        c1 = np.zeros(r * cc)
        c2 = np.zeros(r * cc)
        self.lib.ozo_accumulate(_ptr(flat), r * cc, C.byref(c), _ptr(c1), _ptr(c2))
        return c1.reshape(cc, r).T, c2.reshape(cc, r).T

    def crt_reduce(self, c1, c2, n_moduli, prec=0):
        c = self.constants(n_moduli, prec)
        f = np.vectorize(lambda x, y: self.lib.ozo_crt_reduce_element(float(x), float(y), C.byref(c)))
        return f(c1, c2).astype(np.float64)

    def unscale(self, cpp, mu_exp, nu_exp):
        cpp = _f(cpp, np.float64)
        m, n = cpp.shape
        mu = np.ascontiguousarray(mu_exp, np.int32)
        nu = np.ascontiguousarray(nu_exp, np.int32)
        out = np.zeros((m, n), order="F")
        self.lib.ozo_unscale(_ptr(cpp), m, n, _ptr(mu), _ptr(nu), _ptr(out))
        return out

    # -- pipeline --------------------------------------------------------------------
    def gemm(self, a, b, n_moduli, mode, prec=0, block_k=1 << 17):
        dt = np.float64 if prec == 0 else np.float32
        a, b = _f(a, dt), _f(b, dt)
        m, k = a.shape
        n = b.shape[1]
        c = np.zeros((m, n), np.float64, order="F")
        fn = self.lib.ozo_gemm_f64 if prec == 0 else self.lib.ozo_gemm_f32
        st = fn(_ptr(a), _ptr(b), m, n, k, n_moduli, mode, block_k, _ptr(c))
        if st == 1:
            raise ValueError("ConfigError")
        if st == 2:
            raise ValueError("InputError")
        return c

    def gemm_consts(self, a, b, consts: Constants, mode, block_k=1 << 17):
        a, b = _f(a, np.float64), _f(b, np.float64)
        m, k = a.shape
        n = b.shape[1]
        c = np.zeros((m, n), np.float64, order="F")
        st = self.lib.ozo_gemm_f64_consts(_ptr(a), _ptr(b), m, n, k, C.byref(consts), mode, block_k, _ptr(c))
        if st:
            raise ValueError(f"status {st}")
        return c

    def gemm_scaled(self, a, b, n_moduli, mu_exp, nu_exp, block_k=1 << 17, prec=0):
        """the pipeline after scaling, with given exponents: entry (i, j) depends only on
        row i of a, column j of b, mu_exp[i], nu_exp[j] -- so sampled rows/columns of a
        large problem reproduce those entries of its C exactly"""
        dt = np.float64 if prec == 0 else np.float32
        a, b = _f(a, dt), _f(b, dt)
        m, k = a.shape
        n = b.shape[1]
        cs = self.constants(n_moduli, prec)
        mu = np.ascontiguousarray(mu_exp, np.int32)
        nu = np.ascontiguousarray(nu_exp, np.int32)
        c = np.zeros((m, n), np.float64, order="F")
        fn = self.lib.ozo_gemm_f64_scaled if prec == 0 else self.lib.ozo_gemm_f32_scaled
        fn(_ptr(a), _ptr(b), m, n, k, C.byref(cs), _ptr(mu), _ptr(nu), block_k, _ptr(c))
        return c

    def accurate_exponent(self, cmax: int, base: int, n_moduli: int) -> int:
        return self.lib.ozo_accurate_exponent(int(cmax), int(base), C.byref(self.constants(n_moduli)))

    def products_u8(self, a, b, n_moduli, mode, block_k=1 << 17):
        a, b = _f(a, np.float64), _f(b, np.float64)
        m, k = a.shape
        n = b.shape[1]
        u = np.zeros((n_moduli, n, m), np.uint8)
        st = self.lib.ozo_products_u8_f64(_ptr(a), _ptr(b), m, n, k, n_moduli, mode, block_k, _ptr(u))
        if st:
            raise ValueError(f"status {st}")
        return u.transpose(0, 2, 1)


class RefLib:
    """The unmodified reference (oracle/_ref/libcrtgemm_ref.so)."""

    def __init__(self, path: str = REF_SO):
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_constants.argtypes = [C.c_int, C.c_int] + [_p] * 11
        for nm in ("ref_gemm_f64", "ref_gemm_f32"):
            getattr(L, nm).argtypes = [_i64, _i64, _i64, _p, _p, C.c_int, C.c_int, C.c_int, _i64, C.c_int, _p]
        for nm in ("ref_gemm_tbl_f64", "ref_gemm_tbl_f32"):
            getattr(L, nm).argtypes = [_i64, _i64, _i64, _p, _p, C.c_int, C.c_int, C.c_int, C.c_int, _i64, C.c_int, _p]
        for nm in ("ref_scale_f64", "ref_scale_f32"):
            getattr(L, nm).argtypes = [_i64, _i64, _i64, _p, _p, C.c_int, C.c_int, C.c_int, _i64, C.c_int, _p, _p]
        for nm in ("ref_residues_f64", "ref_residues_f32"):
            getattr(L, nm).argtypes = [_i64, _i64, _p, _p, C.c_int, C.c_int, C.c_int, _p, _p]
        for nm in ("ref_rmod_fast_f64", "ref_rmod_fast_f32"):
            getattr(L, nm).argtypes = [_p, _i64, C.c_int, C.c_int, _p]
        L.ref_mod_u8.argtypes = [_p, _i64, C.c_int32, C.c_int32, _p]
        L.ref_int8_gemm.argtypes = [_i64, _i64, _i64, _p, _p, C.c_int, C.c_int, _p]
        L.ref_accumulate.argtypes = [C.c_int, C.c_int, _i64, _i64, _p, _p, _p]
        L.ref_crt_reduce.argtypes = [C.c_int, C.c_int, _i64, _p, _p, _p]
        L.ref_unscale.argtypes = [C.c_int, C.c_int, _i64, _i64, _p, _p, _p, _p]
        for nm in ("ref_exact_compare_f64", "ref_exact_compare_f32"):
            getattr(L, nm).argtypes = [_i64, _i64, _i64, _p, _p, _p, _p]
        for nm in ("ref_exact_rounded_f64", "ref_exact_rounded_f32"):
            getattr(L, nm).argtypes = [_i64, _i64, _i64, _p, _p, _p]
        L.ref_plain_gemm_f64.argtypes = [_i64, _i64, _i64, _p, _p, _p]
        L.ref_plain_gemm_f32.argtypes = [_i64, _i64, _i64, _p, _p, _p]
        L.ref_dump_tables_csv.argtypes = [C.c_int, C.c_int, C.c_char_p, C.c_int]

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def _check(self, st):
        if st:
            raise ValueError(f"reference status {st}: {self.lib.ref_last_error().decode()}")

    def constants(self, n, prec=0) -> dict:
        mod = np.zeros(20, np.int32)
        q = np.zeros(20, np.int64)
        beta = np.zeros(20, np.int32)
        pp3 = np.zeros(3)
        pp = np.zeros(2, np.float32)
        s1 = np.zeros(20)
        s2 = np.zeros(20)
        p64 = np.zeros(20)
        p32 = np.zeros(20, np.float32)
        mh = np.zeros(20, np.int32)
        pb = C.c_int(0)
        self._check(self.lib.ref_constants(n, prec, *[_ptr(x) for x in (mod, q, beta, pp3, pp, s1, s2, p64, p32, mh)],
                                           C.addressof(pb)))
        return {
            "moduli": mod[:n].tolist(), "q": q[:n].tolist(), "beta": beta[:n].tolist(),
            "P1": pp3[0], "P2": pp3[1], "P_inv": pp3[2], "pp_fast": pp[0], "pp_accu": pp[1],
            "s1": s1[:n].tolist(), "s2": s2[:n].tolist(), "pinv64": p64[:n].tolist(),
            "pinv32": [np.float32(x) for x in p32[:n]], "pinv_mulhi": mh[:n].tolist(), "P_bits": pb.value,
        }

    def tables_csv(self, n, prec=0) -> str:
        buf = C.create_string_buffer(8192)
        self._check(self.lib.ref_dump_tables_csv(n, prec, buf, 8192))
        return buf.value.decode()

    def gemm(self, a, b, n_moduli, mode, prec=0, block_k=1 << 17, threads=1, in_prec=None):
        in_prec = prec if in_prec is None else in_prec
        dt = np.float64 if in_prec == 0 else np.float32
        a, b = _f(a, dt), _f(b, dt)
        m, k = a.shape
        n = b.shape[1]
        c = np.zeros((m, n), np.float64, order="F")
        fn = self.lib.ref_gemm_f64 if in_prec == 0 else self.lib.ref_gemm_f32
        self._check(fn(m, n, k, _ptr(a), _ptr(b), n_moduli, mode, prec, block_k, threads, _ptr(c)))
        return c

    def gemm_tables(self, a, b, n_moduli, mode, prec, table_prec, block_k=1 << 17, threads=1):
        """gemm_emulated(a, b, cfg, build_constants(n, table_prec)) with cfg.precision = prec
        (emulator.hpp:29-32); a/b keep their dtype (float64 or float32)"""
        fn = self.lib.ref_gemm_tbl_f32 if a.dtype == np.float32 else self.lib.ref_gemm_tbl_f64
        a, b = _f(a, a.dtype), _f(b, b.dtype)
        m, k = a.shape
        n = b.shape[1]
        c = np.zeros((m, n), np.float64, order="F")
        self._check(fn(m, n, k, _ptr(a), _ptr(b), n_moduli, mode, prec, table_prec, block_k, threads, _ptr(c)))
        return c

    def scale(self, a, b, n_moduli, mode, prec=0, block_k=1 << 17, threads=1):
        dt = np.float64 if prec == 0 else np.float32
        a, b = _f(a, dt), _f(b, dt)
        m, k = a.shape
        n = b.shape[1]
        mu = np.zeros(m)
        nu = np.zeros(n)
        fn = self.lib.ref_scale_f64 if prec == 0 else self.lib.ref_scale_f32
        self._check(fn(m, n, k, _ptr(a), _ptr(b), n_moduli, mode, prec, block_k, threads, _ptr(mu), _ptr(nu)))
        return mu, nu

    def residues(self, x, scale, side, n_moduli, prec=0):
        dt = np.float64 if prec == 0 else np.float32
        x = _f(x, dt)
        r, c = x.shape
        sc = np.ascontiguousarray(scale, np.float64)
        tr = np.zeros_like(x, order="F")
        planes = np.zeros((n_moduli, c, r), np.int8)
        fn = self.lib.ref_residues_f64 if prec == 0 else self.lib.ref_residues_f32
        self._check(fn(r, c, _ptr(x), _ptr(sc), side, n_moduli, prec, _ptr(tr), _ptr(planes)))
        return tr, planes.transpose(0, 2, 1)

    def int8_gemm(self, a, b, threads=1, use_reference=False):
        a, b = _f(a, np.int8), _f(b, np.int8)
        m, k = a.shape
        n = b.shape[1]
        c = np.zeros((m, n), np.int32, order="F")
        self._check(self.lib.ref_int8_gemm(m, n, k, _ptr(a), _ptr(b), threads, int(use_reference), _ptr(c)))
        return c

    def exact_compare(self, a, b, c, prec=0):
        dt = np.float64 if prec == 0 else np.float32
        a, b = _f(a, dt), _f(b, dt)
        c = _f(c, np.float64)
        m, k = a.shape
        n = b.shape[1]
        rep = np.zeros(3)
        fn = self.lib.ref_exact_compare_f64 if prec == 0 else self.lib.ref_exact_compare_f32
        self._check(fn(m, n, k, _ptr(a), _ptr(b), _ptr(c), _ptr(rep)))
        return {"max_rel_err": rep[0], "median_rel_err": rep[1], "exact_match": bool(rep[2])}

    def exact_rounded(self, a, b, prec=0):
        """the exact product a b (GMP, oracle.cpp exact_gemm), each entry rounded to FP64"""
        dt = np.float64 if prec == 0 else np.float32
        a, b = _f(a, dt), _f(b, dt)
        m, k = a.shape
        n = b.shape[1]
        out = np.zeros((m, n), order="F")
        fn = self.lib.ref_exact_rounded_f64 if prec == 0 else self.lib.ref_exact_rounded_f32
        self._check(fn(m, n, k, _ptr(a), _ptr(b), _ptr(out)))
        return out

    @staticmethod
    def rel_errors(c, rounded_exact):
        """compare()'s componentwise |c - r| / |r| (oracle.cpp:116-157) against
        rounded exact values: 0 where equal, +inf where r = 0 != c"""
        c = np.asarray(c, np.float64)
        r = np.asarray(rounded_exact, np.float64)
        with np.errstate(divide="ignore", invalid="ignore"):
            e = np.abs(c - r) / np.abs(r)
        e = np.where(c == r, 0.0, e)
        return np.where((r == 0) & (c != 0), np.inf, e)

    def plain_gemm(self, a, b, prec=0):
        dt = np.float64 if prec == 0 else np.float32
        a, b = _f(a, dt), _f(b, dt)
        m, k = a.shape
        n = b.shape[1]
        c = np.zeros((m, n), dt, order="F")
        fn = self.lib.ref_plain_gemm_f64 if prec == 0 else self.lib.ref_plain_gemm_f32
        self._check(fn(m, n, k, _ptr(a), _ptr(b), _ptr(c)))
        return c
