"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/ozaki2_b200.h declares (and the C++ crtgemm drop-in), builds
the constant tables on the host exactly like the reference, maps errors like
the reference, and refuses to compute without a B200 (no CPU fallback)."""
import ctypes as C
import json
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2508_03984_b200 import _lib
from paper_2508_03984_b200 import emulator as emu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ozaki2_b200.h")
GOLDEN = os.path.join(ROOT, "tests", "golden")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ozk_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    declared = header_symbols()
    assert set(declared) == set(_lib.EXPORTED_SYMBOLS)
    for name in declared:
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared:
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_cpp_dropin_symbols_exported():
    out = subprocess.run(["nm", "-DC", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for sig in ("crtgemm::gemm_emulated(crtgemm::Matrix<double> const&, crtgemm::Matrix<double> const&, "
                "crtgemm::EmuConfig const&)",
                "crtgemm::gemm_emulated(crtgemm::Matrix<float> const&, crtgemm::Matrix<float> const&, "
                "crtgemm::EmuConfig const&)",
                "crtgemm::build_constants(int, crtgemm::Precision)",
                "crtgemm::select_moduli(int)", "crtgemm::mod_inverse(long, long)",
                "crtgemm::dump_tables_csv", "crtgemm::to_fp32("):
        assert sig in out, sig


def test_sm100a_cubin_and_tcgen05():
    """the library carries sm_100a SASS with tcgen05 int8 MMA, TMA and TMEM loads"""
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for mnem in ("UTCIMMA", "UTMALDG", "LDTM"):
        assert mnem in sass, mnem


def test_constants_match_reference_golden():
    gold = json.load(open(os.path.join(GOLDEN, "constants.json")))
    for key, g in gold.items():
        n, prec = map(int, key.split("_"))
        c = emu.build_constants(n, emu.Precision(prec))
        assert list(c.moduli[:n]) == g["moduli"]
        assert list(c.q[:n]) == g["q"]
        assert list(c.beta[:n]) == g["beta"]
        assert list(c.pinv_mulhi[:n]) == g["pinv_mulhi"]
        assert c.P_bits == g["P_bits"]
        for f in ("P1", "P2", "P_inv", "pp_fast", "pp_accu"):
            assert float(getattr(c, f)) == float.fromhex(g[f]), (key, f)
        for f in ("s1", "s2", "pinv64", "pinv32"):
            assert [float(x) for x in getattr(c, f)[:n]] == [float.fromhex(x) for x in g[f]], (key, f)


def test_tables_csv_matches_reference_dump():
    for n, prec, name in ((14, 0, "tables_14_fp64.csv"), (8, 1, "tables_8_fp32.csv"), (20, 0, "tables_20_fp64.csv")):
        assert emu.dump_tables_csv(emu.build_constants(n, emu.Precision(prec))) == open(
            os.path.join(GOLDEN, name)).read()


def test_big_p_limbs():
    c = emu.build_constants(20)
    P = sum(int(c.P_limbs[i]) << (32 * i) for i in range(6))
    want = 1
    for p in c.moduli[:20]:
        want *= int(p)
    assert P == want and P.bit_length() == c.P_bits


def test_config_errors_like_reference():
    with pytest.raises(emu.ConfigError):
        emu.build_constants(21)
    with pytest.raises(emu.ConfigError):
        emu.build_constants(1)
    with pytest.raises(emu.ConfigError):
        emu.build_constants(19, emu.Precision.Fp32)
    with pytest.raises(emu.ConfigError):
        emu.select_moduli(0)
    with pytest.raises(ArithmeticError):
        emu.mod_inverse(4, 10)
    assert emu.mod_inverse(255, 256) == 255 and emu.mod_inverse(3, 10) == 7
    assert emu.select_moduli(5) == [256, 255, 253, 251, 247]


def test_validation_order_before_device():
    """emulator.cpp:14-18 checks run on the host, before any device work"""
    a = np.zeros((3, 4))
    b = np.zeros((4, 2))
    with pytest.raises(emu.InputError):
        emu.gemm_emulated(a, np.zeros((5, 2)), emu.EmuConfig())
    with pytest.raises(emu.InputError):
        emu.gemm_emulated(np.zeros((0, 4)), b, emu.EmuConfig())
    with pytest.raises(emu.ConfigError):
        emu.gemm_emulated(a, b, emu.EmuConfig(block_k=0))
    with pytest.raises(emu.ConfigError):
        emu.gemm_emulated(a, b, emu.EmuConfig(block_k=(1 << 17) + 1))
    with pytest.raises(emu.ConfigError):
        emu.gemm_emulated(a, b, emu.EmuConfig(threads=0))
    with pytest.raises(emu.ConfigError):  # N range checked first (build_constants)
        emu.gemm_emulated(a, b, emu.EmuConfig(n_moduli=25, threads=0))
    with pytest.raises(emu.ConfigError):  # FP32 inputs need an Fp32 config
        emu.gemm_emulated(a.astype(np.float32), b.astype(np.float32), emu.EmuConfig())


def test_default_config_mirrors_reference():
    cfg = emu.EmuConfig()
    assert (cfg.n_moduli, cfg.mode, cfg.precision, cfg.block_k, cfg.threads) == (
        15, emu.ScaleMode.Fast, emu.Precision.Fp64, 1 << 17, 1)  # emulator.hpp:12-18
    L = _lib.load()
    c = L.ozk_default_config(14, 1, 1)
    assert (c.n_moduli, c.mode, c.precision, c.a_type, c.c_type, c.block_k) == (14, 1, 1, 1, 0, 1 << 17)


def test_no_cpu_fallback():
    """Without a usable B200 the compute entry points fail loudly."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    L = _lib.load()
    h = C.c_void_p()
    assert L.ozk_create(C.byref(h), 0) == _lib.OZK_CUDA_ERROR
    with pytest.raises(_lib.CudaError):
        emu.gemm_emulated(np.ones((2, 2)), np.ones((2, 2)), emu.EmuConfig(n_moduli=4))
