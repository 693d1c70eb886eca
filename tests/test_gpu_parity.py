"""GPU parity: every stage of the CUDA path against the CPU oracle, bit-exact.

Each test calls through the C ABI (paper_2508_03984_b200.Context -> ozk_*),
on cuda:0, and compares with oracle/ozk_oracle.c (the restatement pinned to
the reference in tests/test_oracle.py), or directly with the compiled
reference (oracle/_ref) where noted.
"""
import numpy as np
import pytest

from paper_2508_03984_b200 import EmuConfig, Precision, ScaleMode, gemm_emulated, gen_int_matrix, gen_matrix
from paper_2508_03984_b200 import _lib

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _dev_colmajor(x: np.ndarray):
    """host Fortran array -> CUDA tensor (rows, cols) with stride (1, rows)"""
    t = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
    return t.t()


def _bits(x):
    return np.ascontiguousarray(x).view(np.int64 if x.dtype == np.float64 else np.int32)


def _planes_colmajor(mats, ld):
    """list of (rows x cols) int8 matrices -> [N][cols][ld] column-major device planes"""
    n_mod = len(mats)
    rows, cols = mats[0].shape
    buf = np.zeros((n_mod, cols, ld), np.int8)
    for i, m in enumerate(mats):
        buf[i, :, :rows] = m.T
    return torch.from_numpy(buf).cuda()


SHAPES = [(1, 1, 1), (17, 33, 45), (128, 256, 128), (256, 256, 256), (300, 500, 1000), (513, 260, 2049)]


@pytest.mark.parametrize("m,n,k", SHAPES)
def test_products_int32_and_u8(ctx, oracle, m, n, k):
    rng = np.random.default_rng(m * 1000 + n + k)
    n_mod = 3
    cfg = EmuConfig(n_moduli=n_mod)
    consts = oracle.constants(n_mod)
    A = [rng.integers(-128, 128, size=(m, k), dtype=np.int8) for _ in range(n_mod)]
    B = [rng.integers(-128, 128, size=(k, n), dtype=np.int8) for _ in range(n_mod)]
    pa = _planes_colmajor(A, ctx.plane_ld(m))
    pb = _planes_colmajor(B, ctx.plane_ld(k))
    out = torch.zeros((n_mod, n, m), dtype=torch.int32, device="cuda")
    ctx.stage_products(cfg, m, n, k, pa, pb, _lib.OZK_PRODUCTS_I32, out, m)
    u = torch.zeros((n_mod, n, m), dtype=torch.uint8, device="cuda")
    ctx.stage_products(cfg, m, n, k, pa, pb, _lib.OZK_PRODUCTS_U8, u, m)
    got = out.cpu().numpy()
    got_u = u.cpu().numpy()
    for i in range(n_mod):
        want = oracle.int8_gemm(A[i], B[i])
        np.testing.assert_array_equal(got[i].T, want)
        p, pinv = consts.moduli[i], consts.pinv_mulhi[i]
        want_u = np.vectorize(lambda x: oracle.mod_u8(int(x), p, pinv))(want).astype(np.uint8)
        np.testing.assert_array_equal(got_u[i].T, want_u)


def test_products_wraparound_k_2_17(ctx, oracle):
    """SPEC.md:239 / :493: k = 2^17 all -128 -> 2^31 wraps to INT32_MIN; mod 256 = 0."""
    m, n, k = 4, 4, 1 << 17
    cfg = EmuConfig(n_moduli=2)
    pa = torch.full((2, k, ctx.plane_ld(m)), -128, dtype=torch.int8, device="cuda")
    pb = torch.full((2, n, ctx.plane_ld(k)), -128, dtype=torch.int8, device="cuda")
    out = torch.zeros((2, n, m), dtype=torch.int32, device="cuda")
    ctx.stage_products(cfg, m, n, k, pa, pb, _lib.OZK_PRODUCTS_I32, out, m)
    assert (out == -(2 ** 31)).all()
    u = torch.ones((2, n, m), dtype=torch.uint8, device="cuda")
    ctx.stage_products(cfg, m, n, k, pa, pb, _lib.OZK_PRODUCTS_U8, u, m)
    assert (u[0] == 0).all()  # p = 256
    assert (u[1] == oracle.mod_u8(-(2 ** 31), 255, oracle.constants(2).pinv_mulhi[1])).all()


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("phi", [0.0, 0.5, 2.0, 4.0])
def test_scale_exponents(ctx, oracle, prec, mode, phi):
    m, n, k = 190, 130, 777
    N = 14 if prec == 0 else 8
    dt = np.float64 if prec == 0 else np.float32
    a = gen_matrix(m, k, phi, 11, dt)
    b = gen_matrix(k, n, phi, 12, dt)
    a[5, :] = 0.0  # zero row -> sentinel mu = 1
    b[:, 7] = 0.0
    cfg = EmuConfig(n_moduli=N, mode=ScaleMode(mode), precision=Precision(prec))
    mu = torch.zeros(m, dtype=torch.int32, device="cuda")
    nu = torch.zeros(n, dtype=torch.int32, device="cuda")
    ctx.stage_scale(_dev_colmajor(a), _dev_colmajor(b), cfg, mu, nu)
    wmu, wnu = oracle.scale(a, b, N, mode, prec)
    np.testing.assert_array_equal(mu.cpu().numpy(), wmu)
    np.testing.assert_array_equal(nu.cpu().numpy(), wnu)


@pytest.mark.parametrize("m", [192, 190])  # whole 64-row groups (vectorised rows) and a ragged one
@pytest.mark.parametrize("trans", [False, True])
def test_scale_flagged_lines_exact_path(ctx, oracle, m, trans):
    """Lines the fast budget cannot decide from the parallel sum — here maxima
    outside [2^-400, 2^500) — take the exact sequential recompute inside the
    reduction kernels (the last block of a row group / the column's warp)."""
    n, k = 130, 3000
    a = gen_matrix(m, k, 0.5, 41)
    b = gen_matrix(k, n, 0.5, 42)
    a[[3, 70, m - 1], :] *= 2.0 ** -450
    a[[9, 100], :] *= 2.0 ** 510
    b[:, [0, 64, n - 1]] *= 2.0 ** -450
    b[:, [11]] *= 2.0 ** 505
    cfg = EmuConfig(n_moduli=14, mode=ScaleMode.Fast)
    wmu, wnu = oracle.scale(a, b, 14, 0)
    mu = torch.zeros(m, dtype=torch.int32, device="cuda")
    nu = torch.zeros(n, dtype=torch.int32, device="cuda")
    ctx.stage_scale(_dev_colmajor(a), _dev_colmajor(b), cfg, mu, nu)
    np.testing.assert_array_equal(mu.cpu().numpy(), wmu)
    np.testing.assert_array_equal(nu.cpu().numpy(), wnu)
    want = oracle.gemm(a, b, 14, 0)
    if trans:  # the same lines through the transposed-operand reductions (A^T columns, B^T rows)
        C = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
        ctx.gemm(_dev_colmajor(np.asfortranarray(a.T)), _dev_colmajor(np.asfortranarray(b.T)), cfg, C,
                 trans_a=True, trans_b=True)
        got = C.cpu().numpy()
    else:
        got = gemm_emulated(a, b, cfg).c
    np.testing.assert_array_equal(_bits(got), _bits(want))


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("N", [2, 8, 12, 13, 16, 19, 20])
def test_residue_planes(ctx, oracle, prec, N):
    if prec == 1 and N > 18:
        pytest.skip("fp32 tables stop at N = 18")
    m, n, k = 70, 90, 300
    dt = np.float64 if prec == 0 else np.float32
    a = gen_matrix(m, k, 2.0, 21, dt)
    b = gen_matrix(k, n, 2.0, 22, dt)
    cfg = EmuConfig(n_moduli=N, mode=ScaleMode.Accurate, precision=Precision(prec))
    mu, nu = oracle.scale(a, b, N, 1, prec)
    pa = torch.zeros((N, k, ctx.plane_ld(m)), dtype=torch.int8, device="cuda")
    pb = torch.zeros((N, n, ctx.plane_ld(k)), dtype=torch.int8, device="cuda")
    ctx.stage_residues(_dev_colmajor(a), _dev_colmajor(b), cfg, torch.from_numpy(mu).cuda(),
                       torch.from_numpy(nu).cuda(), pa, pb)
    wa = oracle.residues(oracle.truncate(a, mu, 0, prec), N, prec)  # (N, m, k)
    wb = oracle.residues(oracle.truncate(b, nu, 1, prec), N, prec)  # (N, k, n)
    np.testing.assert_array_equal(pa.cpu().numpy()[:, :, :m].transpose(0, 2, 1), wa)
    np.testing.assert_array_equal(pb.cpu().numpy()[:, :, :k], wb.transpose(0, 2, 1))


@pytest.mark.parametrize("N", [2, 9, 14, 20])
@pytest.mark.parametrize("c_f32", [False, True])
@pytest.mark.parametrize("m,n,pad", [(61, 37, 16), (70, 37, 8), (3000, 5, 16), (129, 6, 16)])
def test_reconstruct(ctx, oracle, N, c_f32, m, n, pad):
    """pad 16: the bulk-copy kernel (several 1024-row tiles and a partial one at
    m = 3000); pad 8 (ldu = 72, not 16-byte aligned): the register-staged fallback"""
    rng = np.random.default_rng(N)
    consts = oracle.constants(N)
    U = np.stack([rng.integers(0, p, size=(m, n)) for p in consts.moduli[:N]]).astype(np.uint8)
    mu = rng.integers(-60, 60, size=m).astype(np.int32)
    nu = rng.integers(-60, 60, size=n).astype(np.int32)
    c1, c2 = oracle.accumulate(U, N)
    want = oracle.unscale(oracle.crt_reduce(c1, c2, N), mu, nu)
    ldu = (m + pad - 1) // pad * pad
    Ud = np.zeros((N, n, ldu), np.uint8)
    Ud[:, :, :m] = U.transpose(0, 2, 1)
    cdt = torch.float32 if c_f32 else torch.float64
    Cd = torch.zeros((n, m), dtype=cdt, device="cuda").t()
    ctx.stage_reconstruct(EmuConfig(n_moduli=N), m, n, torch.from_numpy(Ud).cuda(), ldu,
                          torch.from_numpy(mu).cuda(), torch.from_numpy(nu).cuda(), Cd)
    got = Cd.cpu().numpy()
    if c_f32:
        np.testing.assert_array_equal(got, want.astype(np.float32))
    else:
        np.testing.assert_array_equal(_bits(got), _bits(want))


@pytest.mark.parametrize("N", [9, 14, 20])
@pytest.mark.parametrize("c_f32", [False, True])
@pytest.mark.parametrize("lo,hi", [(-1021, 1021), (500, 530), (-530, -500), (-511, 511)])
def test_reconstruct_unscale_range(ctx, oracle, N, c_f32, lo, hi):
    """unscale (reconstruct.cpp:49-69) across the exponent range: results that
    are subnormal, overflow to inf, or leave the range of the fast unscale
    (|mu|, |nu| > 511 -> 2^-(mu+nu) not a normal double) equal std::ldexp's"""
    rng = np.random.default_rng(N + abs(lo))
    m, n = 300, 41
    consts = oracle.constants(N)
    U = np.stack([rng.integers(0, p, size=(m, n)) for p in consts.moduli[:N]]).astype(np.uint8)
    mu = rng.integers(lo, hi + 1, size=m).astype(np.int32)
    nu = rng.integers(lo, hi + 1, size=n).astype(np.int32)
    c1, c2 = oracle.accumulate(U, N)
    want = oracle.unscale(oracle.crt_reduce(c1, c2, N), mu, nu)
    ldu = (m + 15) // 16 * 16
    Ud = np.zeros((N, n, ldu), np.uint8)
    Ud[:, :, :m] = U.transpose(0, 2, 1)
    cdt = torch.float32 if c_f32 else torch.float64
    Cd = torch.zeros((n, m), dtype=cdt, device="cuda").t()
    ctx.stage_reconstruct(EmuConfig(n_moduli=N), m, n, torch.from_numpy(Ud).cuda(), ldu,
                          torch.from_numpy(mu).cuda(), torch.from_numpy(nu).cuda(), Cd)
    got = Cd.cpu().numpy()
    if c_f32:
        with np.errstate(over="ignore"):
            np.testing.assert_array_equal(got, want.astype(np.float32))
    else:
        np.testing.assert_array_equal(_bits(got), _bits(want))
    if lo == -1021 and not c_f32:
        fin = want[np.isfinite(want) & (want != 0)]
        assert (np.abs(fin) < 2.2250738585072014e-308).any() and np.isinf(want).any()


GEMM_CASES = [
    (64, 64, 64, 0.5, 14),
    (100, 130, 257, 0.0, 14),
    (257, 129, 1000, 0.5, 12),
    (300, 300, 300, 2.0, 16),
    (33, 500, 4000, 1.0, 20),
    (520, 260, 130, 4.0, 17),
    (1, 1, 1, 0.5, 2),
]


@pytest.mark.parametrize("m,n,k,phi,N", GEMM_CASES)
@pytest.mark.parametrize("mode", [ScaleMode.Fast, ScaleMode.Accurate])
def test_gemm_fp64_bitexact(oracle, m, n, k, phi, N, mode):
    a = gen_matrix(m, k, phi, 1)
    b = gen_matrix(k, n, phi, 2)
    got = gemm_emulated(a, b, EmuConfig(n_moduli=N, mode=mode)).c
    want = oracle.gemm(a, b, N, int(mode))
    np.testing.assert_array_equal(_bits(got), _bits(want))


@pytest.mark.parametrize("m,n,k,phi,N", [(64, 64, 64, 0.5, 8), (200, 150, 700, 1.0, 6), (129, 257, 513, 0.5, 18)])
@pytest.mark.parametrize("mode", [ScaleMode.Fast, ScaleMode.Accurate])
@pytest.mark.parametrize("f32_inputs", [True, False])
def test_gemm_fp32_bitexact(oracle, m, n, k, phi, N, mode, f32_inputs):
    a = gen_matrix(m, k, phi, 3)
    b = gen_matrix(k, n, phi, 4)
    cfg = EmuConfig(n_moduli=N, mode=mode, precision=Precision.Fp32)
    if f32_inputs:
        a, b = a.astype(np.float32), b.astype(np.float32)
    got = gemm_emulated(a, b, cfg).c
    want = oracle.gemm(a.astype(np.float32), b.astype(np.float32), N, int(mode), prec=1)
    np.testing.assert_array_equal(_bits(got), _bits(want))


def test_gemm_matches_compiled_reference(ref):
    """Direct cross-check against the unmodified reference (oracle/_ref)."""
    a = gen_matrix(150, 700, 0.5, 5)
    b = gen_matrix(700, 90, 0.5, 6)
    for mode in (ScaleMode.Fast, ScaleMode.Accurate):
        got = gemm_emulated(a, b, EmuConfig(n_moduli=15, mode=mode)).c
        want = ref.gemm(a, b, 15, int(mode))
        np.testing.assert_array_equal(_bits(got), _bits(want))


def test_integer_exactness(oracle):
    """SPEC.md:357 (B = I, small-integer A, N = 15, accurate). The reference
    itself is not exact here (1-ulp misses, e.g. -1 -> -0.9999999999999999);
    the GPU must reproduce it bit-for-bit and stay within 2 ulp of A."""
    a = gen_int_matrix(50, 50, 100, seed=7)
    b = np.asfortranarray(np.eye(50))
    got = gemm_emulated(a, b, EmuConfig(n_moduli=15, mode=ScaleMode.Accurate)).c
    np.testing.assert_array_equal(_bits(got), _bits(oracle.gemm(a, b, 15, 1)))
    assert np.all(np.abs(got - a) <= 2 * np.spacing(np.abs(a) + 1e-300))


@pytest.mark.parametrize("prec,N,lo,hi", [(0, 12, 45, 62), (0, 14, 48, 71), (0, 2, 40, 60), (0, 20, 49, 71),
                                          (1, 3, 18, 30), (1, 8, 35, 43), (1, 4, 20, 40)])
def test_residue_planes_large_magnitudes(ctx, oracle, prec, N, lo, hi):
    """Scaled values straddling the symmetric-residue domain bound (2^50 FP64,
    2^21 / 2^43 FP32) so both the fast and the literal rmod_fast paths run."""
    m, n, k = 40, 36, 200
    dt = np.float64 if prec == 0 else np.float32
    rng = np.random.default_rng(N + 100 * prec)
    a = gen_matrix(m, k, 0.0, 31, dt)
    b = gen_matrix(k, n, 0.0, 32, dt)
    mu = rng.integers(lo, hi, size=m).astype(np.int32)
    nu = rng.integers(lo, hi, size=n).astype(np.int32)
    cfg = EmuConfig(n_moduli=N, mode=ScaleMode.Fast, precision=Precision(prec))
    pa = torch.zeros((N, k, ctx.plane_ld(m)), dtype=torch.int8, device="cuda")
    pb = torch.zeros((N, n, ctx.plane_ld(k)), dtype=torch.int8, device="cuda")
    ctx.stage_residues(_dev_colmajor(a), _dev_colmajor(b), cfg, torch.from_numpy(mu).cuda(),
                       torch.from_numpy(nu).cuda(), pa, pb)
    wa = oracle.residues(oracle.truncate(a, mu, 0, prec), N, prec)
    wb = oracle.residues(oracle.truncate(b, nu, 1, prec), N, prec)
    np.testing.assert_array_equal(pa.cpu().numpy()[:, :, :m].transpose(0, 2, 1), wa)
    np.testing.assert_array_equal(pb.cpu().numpy()[:, :, :k], wb.transpose(0, 2, 1))


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_nonfinite_is_input_error(bad):
    """emulator.cpp:19-22: NaN/Inf anywhere in A or B -> InputError."""
    from paper_2508_03984_b200 import InputError

    a = gen_matrix(30, 40, 0.5, 1)
    b = gen_matrix(40, 20, 0.5, 2)
    a2 = a.copy()
    a2[7, 11] = bad
    with pytest.raises(InputError):
        gemm_emulated(a2, b, EmuConfig(n_moduli=8))
    b2 = b.copy()
    b2[39, 19] = bad
    with pytest.raises(InputError):
        gemm_emulated(a, b2, EmuConfig(n_moduli=8, mode=ScaleMode.Accurate))
    gemm_emulated(a, b, EmuConfig(n_moduli=8))  # the handle recovers


def test_huge_finite_inputs(oracle):
    """entries near the top of the FP64 range are legal (no false non-finite)"""
    a = gen_matrix(20, 30, 1.0, 5) * 1e300
    b = gen_matrix(30, 10, 1.0, 6) * 1e-300
    for mode in (ScaleMode.Fast, ScaleMode.Accurate):
        got = gemm_emulated(a, b, EmuConfig(n_moduli=14, mode=mode)).c
        np.testing.assert_array_equal(_bits(got), _bits(oracle.gemm(a, b, 14, int(mode))))


def test_zero_matrix_and_alpha_beta(ctx, oracle):
    """zero inputs give exact zeros; alpha/beta extension applied in FP64"""
    m, n, k = 64, 48, 80
    a = gen_matrix(m, k, 0.5, 8)
    b = gen_matrix(k, n, 0.5, 9)
    A, B = _dev_colmajor(a), _dev_colmajor(b)
    C0 = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
    cfg = EmuConfig(n_moduli=14)
    ctx.gemm(A, B, cfg, C0)
    base = C0.cpu().numpy()
    np.testing.assert_array_equal(_bits(base), _bits(oracle.gemm(a, b, 14, 0)))
    Cin = torch.from_numpy(np.ascontiguousarray(gen_matrix(m, n, 0.5, 10).T)).cuda().t()
    want = 2.5 * base + (-0.75) * Cin.cpu().numpy()
    ctx.gemm(A, B, cfg, Cin, alpha=2.5, beta=-0.75)
    np.testing.assert_array_equal(_bits(Cin.cpu().numpy()), _bits(want))
    Z = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
    ctx.gemm(_dev_colmajor(np.zeros((m, k))), B, cfg, Z)
    assert (Z == 0).all()


@pytest.mark.parametrize("mode", [ScaleMode.Fast, ScaleMode.Accurate])
@pytest.mark.parametrize("prec", [Precision.Fp64, Precision.Fp32])
def test_host_pipeline_multiblock(oracle, mode, prec):
    """ozk_gemm_host splits B/C into column blocks (H2D/D2H overlapped with
    compute); results must equal the unblocked reference exactly."""
    m, n, k = 260, 2600, 333
    a = gen_matrix(m, k, 1.0, 41)
    b = gen_matrix(k, n, 1.0, 42)
    N = 14 if prec == Precision.Fp64 else 8
    got = gemm_emulated(a, b, EmuConfig(n_moduli=N, mode=mode, precision=prec)).c
    want = oracle.gemm(a.astype(np.float32) if prec else a, b.astype(np.float32) if prec else b, N, int(mode),
                       prec=int(prec))
    np.testing.assert_array_equal(_bits(got), _bits(want))


def test_host_pipeline_alpha_beta_multiblock(ctx, oracle):
    m, n, k = 100, 2100, 64
    a = gen_matrix(m, k, 0.5, 51)
    b = gen_matrix(k, n, 0.5, 52)
    c0 = gen_matrix(m, n, 0.5, 53)
    base = oracle.gemm(a, b, 12, 0)
    out = np.asfortranarray(c0.copy())
    ctx.gemm_host(a, b, EmuConfig(n_moduli=12), alpha=-1.5, beta=0.25, c=out)
    np.testing.assert_array_equal(_bits(out), _bits(-1.5 * base + 0.25 * c0))


@pytest.mark.parametrize("k,mode", [((1 << 17) + 1000, ScaleMode.Fast), (300000, ScaleMode.Fast),
                                    (200000, ScaleMode.Accurate), (1 << 17, ScaleMode.Accurate)])
def test_long_k_blocked_path(oracle, k, mode):
    """k > 2^17: the reference blocks the inner dimension (emulator.cpp:57-73);
    the GPU chunks K2 by 2^17 and re-reduces the residues. Bit-exact either way."""
    m, n = 9, 7
    a = gen_matrix(m, k, 0.5, 61)
    b = gen_matrix(k, n, 0.5, 62)
    for bk in (1 << 17, 50000):
        got = gemm_emulated(a, b, EmuConfig(n_moduli=14, mode=mode, block_k=bk)).c
        want = oracle.gemm(a, b, 14, int(mode), block_k=bk)
        np.testing.assert_array_equal(_bits(got), _bits(want))


@pytest.mark.parametrize("k", [1 << 19, (1 << 19) + 1000, (1 << 20) + 17])
def test_accurate_long_k_int64_bound(oracle, k):
    """accurate mode beyond k = 2^19: entries of the bound product Abar*Bbar reach
    64*64*k > 2^31, so it accumulates in int64 (scaling.cpp:118-148 keeps it in
    int64 too). Near-2 entries make every Abar/Bbar entry 64: the row maxima are
    exactly 4096*k."""
    m, n = 5, 3
    rng = np.random.default_rng(k)
    a = np.asfortranarray(1.99 - 0.01 * rng.random((m, k)))
    b = np.asfortranarray(1.99 - 0.01 * rng.random((k, n)))
    b[:, 1] = gen_matrix(k, 1, 0.5, 3)[:, 0]
    got = gemm_emulated(a, b, EmuConfig(n_moduli=14, mode=ScaleMode.Accurate)).c
    np.testing.assert_array_equal(_bits(got), _bits(oracle.gemm(a, b, 14, 1)))


def test_shard_accurate_long_k_rejected(ctx):
    from paper_2508_03984_b200 import InputError

    k = (1 << 19) + 1
    A = _dev_colmajor(np.zeros((2, k)))
    B = _dev_colmajor(np.zeros((k, 2)))
    with pytest.raises(InputError):
        ctx.shard_begin(A, B, EmuConfig(n_moduli=8, mode=ScaleMode.Accurate))


@pytest.mark.parametrize("mode", [ScaleMode.Fast, ScaleMode.Accurate])
@pytest.mark.parametrize("m,n,k", [(70, 50, 90), (2100, 2060, 64)])
def test_host_leading_dimensions(ctx, oracle, mode, m, n, k):
    """ozk_gemm_host on BLAS submatrix views (lda > m, ldb > k, ldc > m): the
    result equals the oracle and the rows of C past m are never written (the
    second shape takes the streamed fast-mode pipeline)."""
    a = gen_matrix(m, k, 0.5, 81)
    b = gen_matrix(k, n, 0.5, 82)
    A = np.full((m + 7, k), 7.5, order="F")
    A[:m] = a
    B = np.full((k + 5, n), -3.5, order="F")
    B[:k] = b
    Cbig = np.full((m + 3, n), 123.25, order="F")
    ctx.gemm_host(A[:m], B[:k], EmuConfig(n_moduli=14, mode=mode), c=Cbig[:m])
    np.testing.assert_array_equal(_bits(np.asfortranarray(Cbig[:m])), _bits(oracle.gemm(a, b, 14, int(mode))))
    assert (Cbig[m:] == 123.25).all()


@pytest.mark.parametrize("trans", [False, True])
def test_host_leading_dimensions_alpha_beta(ctx, trans):
    """the column pipeline (beta != 0, transposes) on submatrix views equals
    the same call on dense copies, and leaves C's padding rows alone"""
    m, n, k = 300, 260, 130
    a = gen_matrix(m, k, 0.5, 83)
    b = gen_matrix(k, n, 0.5, 84)
    c0 = gen_matrix(m, n, 0.0, 85)
    sa = np.asfortranarray(a.T) if trans else a  # stored operand
    A = np.full((sa.shape[0] + 9, sa.shape[1]), 1.0, order="F")
    A[:sa.shape[0]] = sa
    B = np.full((k + 3, n), 2.0, order="F")
    B[:k] = b
    Cbig = np.full((m + 5, n), -1.0, order="F")
    Cbig[:m] = c0
    cfg = EmuConfig(n_moduli=14)
    ctx.gemm_host(A[:sa.shape[0]], B[:k], cfg, alpha=1.5, beta=-0.5, c=Cbig[:m], trans_a=trans)
    want = ctx.gemm_host(np.asfortranarray(sa), b, cfg, alpha=1.5, beta=-0.5, c=np.asfortranarray(c0.copy()),
                         trans_a=trans)
    np.testing.assert_array_equal(_bits(np.asfortranarray(Cbig[:m])), _bits(want))
    assert (Cbig[m:] == -1.0).all()


@pytest.mark.parametrize("in_dt,prec,table_prec", [(np.float64, Precision.Fp64, Precision.Fp32),
                                                   (np.float64, Precision.Fp32, Precision.Fp64),
                                                   (np.float32, Precision.Fp32, Precision.Fp64)])
@pytest.mark.parametrize("mode", [ScaleMode.Fast, ScaleMode.Accurate])
def test_config_precision_vs_table_precision(in_dt, prec, table_prec, mode):
    """the explicit-constants overloads (emulator.hpp:29-32) with a table of the
    other precision: cfg.precision decides the FP32 rounding and the FP32-input
    check (emulator.cpp:84-99), the table the arithmetic; equal to the reference."""
    from paper_2508_03984_b200 import build_constants
    from _oracle import RefLib

    if not RefLib.available():
        pytest.skip("oracle/_ref not built")
    ref = RefLib()
    a = gen_matrix(90, 400, 1.0, 86).astype(in_dt)
    b = gen_matrix(400, 70, 1.0, 87).astype(in_dt)
    for N in (8, 10):
        cs = build_constants(N, table_prec)
        got = gemm_emulated(a, b, EmuConfig(n_moduli=N, mode=mode, precision=prec), constants=cs).c
        want = ref.gemm_tables(a, b, N, int(mode), int(prec), int(table_prec))
        np.testing.assert_array_equal(_bits(got), _bits(want))


@pytest.mark.parametrize("m,n,k,prec,c32", [(2050, 2600, 77, Precision.Fp64, False),
                                            (4096, 2048, 300, Precision.Fp64, True),
                                            (2304, 3000, 129, Precision.Fp32, False)])
def test_host_streamed_path(ctx, m, n, k, prec, c32):
    """ozk_gemm_host's streamed fast-mode path (A row blocks and B column blocks
    alternate on the copy stream, C leaves region by region) equals the device
    call bit for bit; the device call is the oracle-pinned one."""
    dt = np.float32 if prec == Precision.Fp32 else np.float64
    a = gen_matrix(m, k, 1.0, 71).astype(dt)
    b = gen_matrix(k, n, 1.0, 72).astype(dt)
    b[:, 5] = 0.0
    a[7, :] = 0.0
    cfg = EmuConfig(n_moduli=8 if prec == Precision.Fp32 else 14, precision=prec)
    cdt = np.float32 if c32 else np.float64
    got = ctx.gemm_host(a, b, cfg, c_dtype=cdt)
    Cd = torch.zeros((n, m), dtype=torch.float32 if c32 else torch.float64, device="cuda").t()
    ctx.gemm(_dev_colmajor(a), _dev_colmajor(b), cfg, Cd)
    np.testing.assert_array_equal(_bits(got), _bits(Cd.cpu().numpy()))


def test_host_streamed_matches_oracle(oracle):
    m, n, k = 2100, 2200, 48
    a = gen_matrix(m, k, 0.5, 73)
    b = gen_matrix(k, n, 0.5, 74)
    got = gemm_emulated(a, b, EmuConfig(n_moduli=13)).c
    np.testing.assert_array_equal(_bits(got), _bits(oracle.gemm(a, b, 13, 0)))


@pytest.mark.parametrize("entry", [3, 8, 13])
def test_fault_injection_corrupt_s1_is_located(ctx, oracle, entry):
    """SPEC.md:461 fault injection through the explicit-constants overload
    (emulator.hpp:28-32): one corrupted s1 entry must make the CRT exactness
    check fail, and the stage exports locate it — the residue planes and the
    per-modulus U_i still equal the oracle, only the reconstruction differs.
    (Not entry 0: integer inputs scaled by 2^mu >= 2^8 have all residues mod
    256 equal to 0, so s1[0] never contributes; fast mode is excluded because
    it is inexact on these inputs in the reference too.)"""
    from paper_2508_03984_b200 import build_constants

    N, m, n, k = 14, 48, 40, 64
    a = gen_int_matrix(m, k, 100, seed=17)
    b = gen_int_matrix(k, n, 100, seed=18)
    exact = a @ b  # small integers: the FP64 product is exact
    good = build_constants(N)
    bad = build_constants(N)
    bad.s1[entry] = bad.s1[entry] * (1.0 + 2.0 ** -20)
    A = torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()
    B = torch.from_numpy(np.ascontiguousarray(b.T)).cuda().t()
    cfg = EmuConfig(n_moduli=N, mode=ScaleMode.Accurate)
    C_good = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
    C_bad = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
    ctx.gemm(A, B, cfg, C_good, constants=good)
    ctx.gemm(A, B, cfg, C_bad, constants=bad)
    np.testing.assert_array_equal(C_good.cpu().numpy(), exact)  # the exactness check passes ...
    assert not np.array_equal(C_bad.cpu().numpy(), exact)      # ... and catches the corruption
    # locate it: the products stage (independent of s1) still matches the oracle
    mu = torch.zeros(m, dtype=torch.int32, device="cuda")
    nu = torch.zeros(n, dtype=torch.int32, device="cuda")
    ctx.stage_scale(A, B, cfg, mu, nu)
    pa = torch.zeros((N, k, ctx.plane_ld(m)), dtype=torch.int8, device="cuda")
    pb = torch.zeros((N, n, ctx.plane_ld(k)), dtype=torch.int8, device="cuda")
    ctx.stage_residues(A, B, cfg, mu, nu, pa, pb)
    ldu = (m + 15) // 16 * 16
    U = torch.zeros((N, n, ldu), dtype=torch.uint8, device="cuda")
    ctx.stage_products(cfg, m, n, k, pa, pb, _lib.OZK_PRODUCTS_U8, U, ldu)
    np.testing.assert_array_equal(U.cpu().numpy()[:, :, :m].transpose(0, 2, 1), oracle.products_u8(a, b, N, 1))


@pytest.mark.parametrize("m,n,k,pad", [(1, 1, 1, 0), (17, 33, 45, 3), (300, 129, 1000, 16), (64, 64, 1 << 17, 0)])
def test_int8_gemm_reference_kernel(ctx, oracle, m, n, k, pad):
    """ozk_int8_gemm_reference (int8_engine.cpp:66-80): the CUDA-core triple loop
    against the oracle and against the tensor-core ozk_int8_gemm; padded
    leading dimensions; k = 2^17 of -128 x -128 wraps like the reference."""
    import ctypes as C

    rng = np.random.default_rng(m + 7 * n + k)
    if k == 1 << 17:
        A = np.full((m, k), -128, np.int8)
        B = np.full((k, n), -128, np.int8)
        A[0, :5] = 3
    else:
        A = rng.integers(-128, 128, size=(m, k), dtype=np.int8)
        B = rng.integers(-128, 128, size=(k, n), dtype=np.int8)
    lda, ldb, ldc = m + pad, k + pad, m + pad
    da = torch.zeros((k, lda), dtype=torch.int8, device="cuda")
    da[:, :m] = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    db = torch.zeros((n, ldb), dtype=torch.int8, device="cuda")
    db[:, :k] = torch.from_numpy(np.ascontiguousarray(B.T)).cuda()
    dc = torch.full((n, ldc), 7, dtype=torch.int32, device="cuda")
    L = ctx._lib
    _lib.check(L.ozk_int8_gemm_reference(ctx.handle, m, n, k, C.c_void_p(da.data_ptr()), lda,
                                         C.c_void_p(db.data_ptr()), ldb, C.c_void_p(dc.data_ptr()), ldc))
    got = dc.cpu().numpy()
    want = oracle.int8_gemm(A, B)
    np.testing.assert_array_equal(got[:, :m].T, want)
    assert (got[:, m:] == 7).all()  # padding rows untouched
    if lda % 16 == 0 and ldb % 16 == 0:
        tc = torch.zeros((n, m), dtype=torch.int32, device="cuda")
        _lib.check(L.ozk_int8_gemm(ctx.handle, m, n, k, C.c_void_p(da.data_ptr()), lda, C.c_void_p(db.data_ptr()),
                                   ldb, C.c_void_p(tc.data_ptr()), m))
        np.testing.assert_array_equal(tc.cpu().numpy(), got[:, :m])


def _pinned_like(x):
    """a page-locked copy of a column-major host array (numpy view of pinned torch memory)"""
    t = torch.empty(x.size, dtype=torch.float64 if x.dtype == np.float64 else torch.float32, pin_memory=True)
    out = t.numpy().reshape(x.shape[::-1]).T  # column-major view
    out[...] = x
    return out, t


@pytest.mark.parametrize("mode", [ScaleMode.Fast, ScaleMode.Accurate])
@pytest.mark.parametrize("beta,c32,trans", [(0.0, False, False), (-0.5, False, False), (0.0, True, False),
                                            (0.0, False, True)])
def test_host_pageable_staging_equals_pinned(ctx, mode, beta, c32, trans):
    """ozk_gemm_host with large pageable operands (numpy memory: the pinned
    staging ring of host_stage.cpp) equals the same call on page-locked
    operands (direct DMA), bit for bit; fast mode at these sizes takes the
    row/column streamed pipeline, the other cases the column pipeline"""
    m, n, k = 2304, 2600, 600
    a = gen_matrix(k, m, 0.5, 91) if trans else gen_matrix(m, k, 0.5, 91)  # stored operand
    b = gen_matrix(k, n, 0.5, 92)
    c0 = gen_matrix(m, n, 0.0, 93)
    cdt = np.float32 if c32 else np.float64
    cfg = EmuConfig(n_moduli=14, mode=mode)
    got = np.asfortranarray(c0.astype(cdt))
    ctx.gemm_host(a, b, cfg, alpha=1.0, beta=beta, c=got, trans_a=trans)
    pa, ta = _pinned_like(a)
    pb, tb = _pinned_like(b)
    pc, tc = _pinned_like(np.asfortranarray(c0.astype(cdt)))
    ctx.gemm_host(pa, pb, cfg, alpha=1.0, beta=beta, c=pc, trans_a=trans)
    np.testing.assert_array_equal(got.view(np.int32 if c32 else np.int64), pc.view(np.int32 if c32 else np.int64))


def test_host_pageable_staging_small_slots():
    """the staging ring with 3000-byte slots (columns split into pieces, many
    slot reuses per call), in a child process (the slot size is read once)"""
    import subprocess
    import sys
    import os
    code = r"""
import numpy as np, torch
from paper_2508_03984_b200 import Context, EmuConfig, ScaleMode, gen_matrix
ctx = Context(0)
m, n, k = 2100, 2200, 700
a, b = gen_matrix(m, k, 0.5, 1), gen_matrix(k, n, 0.5, 2)
for mode in (ScaleMode.Fast, ScaleMode.Accurate):
    cfg = EmuConfig(n_moduli=12, mode=mode)
    got = ctx.gemm_host(a, b, cfg)
    A = torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()
    B = torch.from_numpy(np.ascontiguousarray(b.T)).cuda().t()
    C = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
    ctx.gemm(A, B, cfg, C)
    assert np.array_equal(got.view(np.int64), C.cpu().numpy().view(np.int64)), mode
print("ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, OZK_HOST_STAGE_SLOT="3000", PYTHONPATH=root))
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
