"""Pin the oracle restatement (oracle/ozk_oracle.c) before trusting it.

Three independent anchors:
  * the SPEC.md known-answer examples and SURVEY Appendix A tables,
  * tests/golden/ fixtures produced by the unmodified reference (oracle/_ref),
  * oracle/_ref itself on fresh random inputs, where that library is built.
Plus the algebraic invariants the reference's SPEC states (CRT exactness,
exact s1 accumulation, rmod/mod congruence).
"""
import json
import os

import numpy as np
import pytest

from paper_2508_03984_b200.gen import gen_int_matrix, gen_matrix

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def bits(x):
    return np.ascontiguousarray(x).view(np.int64)


# ---------------------------------------------------------------- SPEC KATs
def test_select_moduli_kat(oracle):
    assert oracle.select_moduli(2) == [256, 255]
    assert oracle.select_moduli(4) == [256, 255, 253, 251]
    assert oracle.select_moduli(5) == [256, 255, 253, 251, 247]
    assert oracle.select_moduli(20) == [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199,
                                        197, 193, 191, 181, 179, 173]
    with pytest.raises(ValueError):
        oracle.select_moduli(21)
    with pytest.raises(ValueError):
        oracle.select_moduli(1)


def test_mod_inverse_kat(oracle):
    assert oracle.mod_inverse(255, 256) == 255
    assert oracle.mod_inverse(1, 7) == 1
    assert oracle.mod_inverse(3, 10) == 7
    with pytest.raises(ArithmeticError):
        oracle.mod_inverse(4, 10)


def test_constants_kat(oracle):
    c = oracle.constants(2, 0)
    assert c.P1 == 65280.0 and c.P2 == 0.0
    assert list(c.q[:2]) == [255, 1]
    c32 = oracle.constants(2, 1)
    assert list(c32.s2[:2]) == [0.0, 0.0]
    with pytest.raises(ValueError):
        oracle.constants(19, 1)                  # fp32 tables stop at 18
    with pytest.raises(ValueError):
        oracle.constants(21, 0)


def test_appendix_a_tables(oracle):
    """SURVEY Appendix A (values read off the reference build)."""
    rows = {8: (64, "0x1.7d690b03a3244p+63", "0x1p+8", "0x1.57a6a12c3f24ap-64", 30.287600, 31.287600),
            12: (95, "0x1.bec64ef0faa26p+94", "0x1.dc188f89p+40", "0x1.255fb5199b04p-95", 45.901703, 46.901703),
            14: (111, "0x1.1e3fc471eb44fp+110", "-0x1.1ff7bc8b7298p+53", "0x1.c9e518641aa18p-111", 53.580563,
                 54.580563),
            16: (126, "0x1.4c232965d6663p+125", "-0x1.616c352d64acap+71", "0x1.8aa1c572fa163p-126", 61.187817,
                 62.187817),
            20: (156, "0x1.4b27367819129p+155", "-0x1.595f0ab0d75c5p+98", "0x1.8bce042d07acep-156", 76.185677,
                 77.185677)}
    for n, (pbits, p1, p2, pinv, ppf, ppa) in rows.items():
        c = oracle.constants(n, 0)
        assert c.P_bits == pbits
        assert c.P1 == float.fromhex(p1) and c.P2 == float.fromhex(p2) and c.P_inv == float.fromhex(pinv)
        assert abs(c.pp_fast - ppf) < 1e-5 and abs(c.pp_accu - ppa) < 1e-5
    mh = [16777215, 16843008, 16976154, 17111422, 17388530, 17821440, 17970573, 18433335, 18755314, 18920559,
          19259942, 19792475, 20355294, 21582749, 21801863, 22253715, 22486738, 23729100, 23994229, 24826399]
    assert list(oracle.constants(20, 0).pinv_mulhi[:20]) == mh


def test_tables_csv_golden(oracle):
    for n, prec, name in ((14, 0, "tables_14_fp64.csv"), (8, 1, "tables_8_fp32.csv"), (20, 0, "tables_20_fp64.csv")):
        lines = open(os.path.join(GOLDEN, name)).read().strip().splitlines()[1:]
        c = oracle.constants(n, prec)
        for i, line in enumerate(lines):
            p, q, beta, s1, s2 = line.split(",")
            assert int(p) == c.moduli[i] and int(q) == c.q[i] and int(beta) == c.beta[i]
            assert float.fromhex(s1) == c.s1[i] and float.fromhex(s2) == c.s2[i]


def test_all_constants_golden(oracle):
    gold = json.load(open(os.path.join(GOLDEN, "constants.json")))
    for key, g in gold.items():
        n, prec = map(int, key.split("_"))
        c = oracle.constants(n, prec).as_dict()
        for f in ("moduli", "q", "beta", "pinv_mulhi"):
            assert c[f] == g[f], (key, f)
        assert c["P_bits"] == g["P_bits"]
        for f in ("P1", "P2", "P_inv", "pp_fast", "pp_accu"):
            assert float(c[f]) == float.fromhex(g[f]), (key, f)
        for f in ("s1", "s2", "pinv64", "pinv32"):
            assert [float(x) for x in c[f]] == [float.fromhex(x) for x in g[f]], (key, f)


def test_rmod_kat(oracle):
    c = oracle.constants(14)
    p, p64, p32 = c.moduli[0], c.pinv64[0], c.pinv32[0]
    assert oracle.lib.ozo_rmod_fast_f64(0.0, p, p64, p32, 14) == 0
    assert oracle.lib.ozo_rmod_fast_f64(255.0, p, p64, p32, 14) == -1
    assert oracle.lib.ozo_rmod_fast_f64(128.0, p, p64, p32, 14) == -128  # 128 wraps
    planes = oracle.residues(np.full((1, 1), 65280.0), 2)
    assert planes.ravel().tolist() == [0, 0]
    planes = oracle.residues(np.ones((1, 1)), 20)
    assert planes.ravel().tolist() == [1] * 20


def test_int8_and_mod_kat(oracle):
    c = oracle.int8_gemm(np.array([[127]], np.int8), np.array([[-128]], np.int8))
    assert c[0, 0] == -16256
    cs = oracle.constants(20)
    assert oracle.mod_u8(-1, 255, cs.pinv_mulhi[1]) == 254
    assert oracle.mod_u8(-(2 ** 31), 256, cs.pinv_mulhi[0]) == 0


def test_mod_u8_exhaustive_sample(oracle):
    """SPEC.md:293 (sampled): mod_u8 == exact nonnegative residue."""
    cs = oracle.constants(20)
    rng = np.random.default_rng(0)
    xs = np.concatenate([np.arange(-3000, 3000), rng.integers(-2 ** 31, 2 ** 31, 3000),
                         np.array([-2 ** 31, 2 ** 31 - 1, -2 ** 31 + 1, 2 ** 31 - 2])])
    for i in range(20):
        p, pinv = cs.moduli[i], cs.pinv_mulhi[i]
        for x in xs[:: (7 if i % 2 else 1)]:
            assert oracle.mod_u8(int(x), p, pinv) == int(x) % p


def test_rmod_congruence(oracle):
    """rmod_fast(x) == x (mod p) with a representative in [-128, 127]."""
    rng = np.random.default_rng(1)
    for n, prec, lim in ((12, 0, 2 ** 52), (14, 0, 2 ** 60), (20, 0, 2 ** 71), (4, 1, 2 ** 22), (8, 1, 2 ** 43)):
        c = oracle.constants(n, prec)
        xs = np.trunc(rng.uniform(-lim, lim, 400))
        if prec == 1:
            xs = xs.astype(np.float32)
        planes = oracle.residues(xs.reshape(-1, 1), n, prec)
        for i in range(n):
            p = c.moduli[i]
            for x, r in zip(xs, planes[i].ravel()):
                assert (int(x) - int(r)) % p == 0


def test_accumulation_exact(oracle):
    """SPEC.md:323 / acceptance 4: sum s1_i U_i in FP64 equals the exact sum."""
    from fractions import Fraction

    c = oracle.constants(20)
    rng = np.random.default_rng(2)
    U = np.stack([rng.integers(0, p, size=(8, 8)) for p in c.moduli[:20]]).astype(np.uint8)
    U[:, 0, 0] = np.array(c.moduli[:20]) - 1  # adversarial: all p_i - 1
    c1, _ = oracle.accumulate(U, 20)
    for i in range(8):
        for j in range(8):
            exact = sum(Fraction(c.s1[t]) * int(U[t, i, j]) for t in range(20))
            assert Fraction(c1[i, j]) == exact


# ---------------------------------------------------------------- golden fixtures
def test_golden_gemm_cases(oracle):
    z = np.load(os.path.join(GOLDEN, "gemm_cases.npz"))
    for idx, (m, n, k, phi, N, mode, prec, bk) in enumerate(z["cases"]):
        N, mode, prec, bk = int(N), int(mode), int(prec), int(bk)
        a, b = z[f"case{idx}_a"], z[f"case{idx}_b"]
        mu, nu = oracle.scale(a, b, N, mode, prec, bk)
        np.testing.assert_array_equal(np.exp2(mu.astype(np.float64)), z[f"case{idx}_mu"])
        np.testing.assert_array_equal(np.exp2(nu.astype(np.float64)), z[f"case{idx}_nu"])
        c = oracle.gemm(a, b, N, mode, prec, bk)
        np.testing.assert_array_equal(bits(c), bits(z[f"case{idx}_c"]), err_msg=f"case {idx}")
    np.testing.assert_array_equal(oracle.gemm(z["int_a"], np.asfortranarray(np.eye(10)), 15, 1), z["int_c"])


def test_golden_stage_dump(oracle):
    z = np.load(os.path.join(GOLDEN, "stages_case.npz"))
    a, b = z["a"], z["b"]
    mu, nu = oracle.scale(a, b, 14, 1)
    np.testing.assert_array_equal(np.exp2(mu.astype(np.float64)), z["mu"])
    ta = oracle.truncate(a, mu, 0)
    tb = oracle.truncate(b, nu, 1)
    np.testing.assert_array_equal(ta, z["trunc_a"])
    np.testing.assert_array_equal(tb, z["trunc_b"])
    pa, pb = oracle.residues(ta, 14), oracle.residues(tb, 14)
    np.testing.assert_array_equal(pa, z["planes_a"])
    np.testing.assert_array_equal(pb, z["planes_b"])
    for i in range(14):
        np.testing.assert_array_equal(oracle.int8_gemm(pa[i], pb[i]), z["products"][i])
    np.testing.assert_array_equal(bits(oracle.gemm(a, b, 14, 1)), bits(z["c"]))


# ---------------------------------------------------------------- live reference
@pytest.mark.parametrize("seed", range(6))
def test_oracle_matches_reference_random(oracle, ref, seed):
    rng = np.random.default_rng(100 + seed)
    m, n, k = (int(x) for x in rng.integers(1, 70, 3))
    phi = float(rng.choice([0.0, 0.5, 1.0, 2.0, 4.0]))
    for prec in (0, 1):
        N = int(rng.integers(2, 21 if prec == 0 else 19))
        dt = np.float64 if prec == 0 else np.float32
        a = gen_matrix(m, k, phi, seed * 7 + 1, dt)
        b = gen_matrix(k, n, phi, seed * 7 + 2, dt)
        for mode in (0, 1):
            bk = int(rng.choice([1 << 17, 16, 33]))
            np.testing.assert_array_equal(bits(oracle.gemm(a, b, N, mode, prec, bk)),
                                          bits(ref.gemm(a, b, N, mode, prec, bk)))
            mu, nu = ref.scale(a, b, N, mode, prec, bk)
            omu, onu = oracle.scale(a, b, N, mode, prec, bk)
            np.testing.assert_array_equal(np.exp2(omu.astype(np.float64)), mu)
            np.testing.assert_array_equal(np.exp2(onu.astype(np.float64)), nu)


def test_reference_kernel_engine_threads_and_wrap(ref):
    """int8_gemm == int8_gemm_reference, threads 1 vs 4 identical."""
    rng = np.random.default_rng(5)
    a = rng.integers(-128, 128, (33, 70), dtype=np.int8)
    b = rng.integers(-128, 128, (70, 21), dtype=np.int8)
    c1 = ref.int8_gemm(a, b, threads=1)
    np.testing.assert_array_equal(c1, ref.int8_gemm(a, b, threads=4))
    np.testing.assert_array_equal(c1, ref.int8_gemm(a, b, use_reference=True))


# ---------------------------------------------------------------- exactness property
@pytest.mark.parametrize("N", [2, 5, 10, 15, 20])
def test_crt_exactness_integers(oracle, N):
    """SPEC acceptance 1 (reduced trial count): integer inputs inside the CRT range
    come back exactly (accurate mode, which honours the uniqueness bound)."""
    c = oracle.constants(N)
    rng = np.random.default_rng(N)
    for trial in range(6):
        m, n, k = (int(x) for x in rng.integers(1, 40, 3))
        # entries small enough that the accurate-mode scale is >= 1 (no truncation),
        # which also keeps 2 sum |a||b| far below P
        g = int(np.floor(0.5 * np.log2(float(c.P1)) - 0.51 * np.log2(k) - 4.6))
        bound = int(2 ** min(max(g, 0), 20))
        a = gen_int_matrix(m, k, bound, seed=trial * 2 + 1)
        b = gen_int_matrix(k, n, bound, seed=trial * 2 + 2)
        want = a.astype(object) @ b.astype(object)
        got = oracle.gemm(a, b, N, 1)
        ok = np.vectorize(lambda g, w: int(g) == w if abs(w) < 2 ** 53 else True)(got, want)
        assert ok.all(), (N, trial)


# ---------------------------------------------------------------- symmetric-residue domain
def _symmetric(x: int, p: int) -> int:
    r = x % p
    if r > p // 2 or (p % 2 == 0 and r == p // 2 and False):
        r -= p
    return ((r + 128) % 256) - 128  # int8 view (p = 256: +-128 -> -128)


@pytest.mark.parametrize("n,prec,lim", [(2, 0, 2 ** 50), (12, 0, 2 ** 50), (14, 0, 2 ** 50), (20, 0, 2 ** 50),
                                        (3, 1, 2 ** 21), (5, 1, 2 ** 43), (8, 1, 2 ** 43), (18, 1, 2 ** 43)])
def test_rmod_fast_is_symmetric_in_domain(oracle, n, prec, lim):
    """The claim behind the GPU's conversion-free residues (ozk_device.cuh):
    inside |x| <= 2^50 (FP64) / the FP32 bounds, rmod_fast returns the
    symmetric residue. Checked on random and near-half-multiple integers."""
    c = oracle.constants(n, prec)
    rng = np.random.default_rng(n * 10 + prec)
    xs = [int(v) for v in rng.integers(-lim, lim, 300, dtype=np.int64)]
    for p in c.moduli[:n]:
        # integers whose quotient by p sits closest to a half-integer, near the bound
        base = (lim // p) * p
        xs += [base - p // 2, base - (p + 1) // 2, -base + p // 2, lim, -lim, lim - 1]
    xs = np.array(xs, dtype=np.float64 if prec == 0 else np.float32)
    planes = oracle.residues(xs.reshape(-1, 1), n, prec)
    for i in range(n):
        p = c.moduli[i]
        for x, r in zip(xs, planes[i].ravel()):
            assert int(r) == _symmetric(int(x), p), (n, prec, p, int(x), int(r))


def test_exact_rounded_reproduces_reference_compare(ref):
    """bench.py's exact-error leg: one exact GEMM (oracle.cpp exact_gemm) rounded
    per entry, then compare()'s error formula in numpy, equals the reference's
    compare() (oracle.cpp:116-157) on the same candidate."""
    from _oracle import RefLib

    from paper_2508_03984_b200 import gen_matrix

    a = gen_matrix(24, 700, 2.0, 41)
    b = gen_matrix(700, 20, 2.0, 42)
    b[:, 3] = 0.0  # exact zeros: error 0 (candidate 0) / inf (candidate != 0)
    ex = ref.exact_rounded(a, b)
    for c in (np.asfortranarray(a @ b), np.asfortranarray(ex.copy())):
        c[0, 3] = 1e-300
        e = RefLib.rel_errors(c, ex)
        rep = ref.exact_compare(a, b, c)
        assert np.isinf(e[0, 3])
        finite = np.isfinite(e)
        e2 = RefLib.rel_errors(np.where(finite, c, 0.0), ex)
        rep2 = ref.exact_compare(a, b, np.asfortranarray(np.where(finite, c, 0.0)))
        assert e2.max() == rep2["max_rel_err"]
        assert np.median(e2) == rep2["median_rel_err"]
        assert rep["max_rel_err"] == np.inf
