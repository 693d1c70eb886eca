"""The C++ drop-in: a program written against the reference's crtgemm API
compiles against include/ and links libozaki2_b200.so (CPU), and on the GPU
produces bit-identical results to the oracle and the reference error contract."""
import os
import subprocess

import numpy as np
import pytest

from paper_2508_03984_b200 import _lib
from paper_2508_03984_b200.gen import gen_matrix

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp")


def build(tmp_path):
    exe = str(tmp_path / "dropin_test")
    libdir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-o", exe,
                    "-L", libdir, "-lozaki2_b200", f"-Wl,-rpath,{libdir}"], check=True,
                   capture_output=True, text=True)
    return exe


def _write(path, x):
    with open(path, "wb") as f:
        np.array(x.shape, np.int64).tofile(f)
        np.asfortranarray(x).T.astype(np.float64).tofile(f)  # column-major payload


def _read(path):
    with open(path, "rb") as f:
        r, c = np.fromfile(f, np.int64, 2)
        return np.fromfile(f, np.float64, r * c).reshape(c, r).T


def test_cpp_dropin_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_cpp_dropin_bitexact(tmp_path, oracle):
    exe = build(tmp_path)
    a = gen_matrix(70, 90, 0.5, 71)
    b = gen_matrix(90, 50, 0.5, 72)
    _write(tmp_path / "a.bin", a)
    _write(tmp_path / "b.bin", b)
    cases = [(14, 0, 0), (14, 1, 0), (16, 1, 0), (8, 0, 1), (7, 1, 1)]
    (tmp_path / "cases.txt").write_text("\n".join(" ".join(map(str, c)) for c in cases))
    out = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True)
    assert out.returncode == 0, (out.returncode, out.stdout, out.stderr)
    for i, (N, mode, prec) in enumerate(cases):
        got = _read(tmp_path / f"c_{i}.bin")
        aa, bb = (a.astype(np.float32), b.astype(np.float32)) if prec else (a, b)
        want = oracle.gemm(aa, bb, N, mode, prec=prec)
        np.testing.assert_array_equal(got.view(np.int64), want.view(np.int64))
    for mode in (0, 1):  # the stage-level API composed by hand == the oracle pipeline
        got = _read(tmp_path / f"stages_{mode}.bin")
        np.testing.assert_array_equal(got.view(np.int64), oracle.gemm(a, b, 14, mode).view(np.int64))
    gold = open(os.path.join(ROOT, "tests", "golden", "tables_14_fp64.csv")).read()
    assert (tmp_path / "tables_14.csv").read_text() == gold


@pytest.mark.gpu
def test_cpp_dropin_large_result(tmp_path):
    """A result above 64 MB takes the drop-in's pre-faulted allocation
    (crtgemm.cpp result_matrix: reserve, huge-page advice, parallel
    MADV_POPULATE_WRITE, then the value-initialising resize): the values must
    equal the C ABI host path's bit for bit, zero padding included."""
    from paper_2508_03984_b200 import EmuConfig, gemm_emulated

    exe = build(tmp_path)
    a = gen_matrix(3000, 160, 0.5, 73)
    b = gen_matrix(160, 3000, 0.5, 74)
    _write(tmp_path / "a.bin", a)
    _write(tmp_path / "b.bin", b)
    (tmp_path / "cases.txt").write_text("14 0 0")
    out = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True)
    assert out.returncode == 0, (out.returncode, out.stdout, out.stderr)
    got = _read(tmp_path / "c_0.bin")
    want = gemm_emulated(a, b, EmuConfig(n_moduli=14)).c
    np.testing.assert_array_equal(got.view(np.int64), want.view(np.int64))
