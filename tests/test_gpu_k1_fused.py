"""GPU parity of the one-pass K1 (csrc/k1_fused.cu): statistics, exponents and
planes of each operand in one read from HBM.

The column kernel is the default for ozk_gemm's contiguous lines of >= 4096
elements (>= 1024 of them) whenever the whole problem is one panel (and for
the accurate-mode bound planes), so the full-size suite runs through it; the
row kernel is opt-in (OZK_K1_FUSED=3). This module runs in-process with the
defaults and again in subprocesses with the kernels taken at every size
(OZK_K1_FUSED_ANY=1, masks 1 and 3: the last test).
These cases aim at the kernels' own boundaries:
the 64-row groups and 128-column slices of the row kernel (ragged rows and
columns, a single slice, many groups), the 512-thread column kernel (columns
shorter and longer than one block pass, lengths off the 8-element vectors),
both operand storages (the row kernel serves A and a transposed B, the
column kernel B and a transposed A), FP32 operands, accurate mode (bound
planes), flagged lines (exact recompute inside the fused finalize), the
self-resetting ticket / accumulator state across many calls of different
shapes on one handle, and non-finite detection. Every result must equal the
oracle bit for bit (reference emulator.cpp:25-78).
"""
import numpy as np
import pytest

from paper_2508_03984_b200 import EmuConfig, InputError, Precision, ScaleMode, gen_matrix

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _bits(x):
    return np.ascontiguousarray(x).view(np.int64 if x.dtype == np.float64 else np.int32)


def _dev(x: np.ndarray, ld: int | None = None):
    """host matrix -> column-major CUDA view with leading dimension ld (NaN padding)"""
    rows, cols = x.shape
    ld = rows if ld is None else ld
    buf = np.full((cols, ld), np.nan, dtype=x.dtype)
    buf[:, :rows] = x.T
    return torch.from_numpy(buf).cuda().t()[:rows]


def _run(ctx, a, b, cfg, ta=False, tb=False, lda=None, ldb=None):
    m, n = a.shape[0], b.shape[1]
    A = _dev(np.asfortranarray(a.T) if ta else a, lda)
    B = _dev(np.asfortranarray(b.T) if tb else b, ldb)
    C = _dev(np.zeros((m, n)))
    ctx.gemm(A, B, cfg, C, trans_a=ta, trans_b=tb)
    return C.cpu().numpy()


# row groups of 64 and column slices of 64 (row kernel); 4096-element block
# passes and 8-element vectors (column kernel)
SHAPES = [(1, 1, 1), (63, 65, 64), (64, 64, 65), (65, 130, 129), (200, 7, 4097), (1000, 300, 8191),
          (2049, 64, 6000), (130, 2050, 1000)]


@pytest.mark.parametrize("m,n,k", SHAPES)
@pytest.mark.parametrize("ta,tb", [(False, False), (True, True)])
@pytest.mark.parametrize("mode", [ScaleMode.Fast, ScaleMode.Accurate])
def test_fused_k1_shapes(ctx, oracle, m, n, k, ta, tb, mode):
    a = gen_matrix(m, k, 1.0, 11 + m)
    b = gen_matrix(k, n, 1.0, 12 + n)
    got = _run(ctx, a, b, EmuConfig(n_moduli=14, mode=mode), ta, tb)
    np.testing.assert_array_equal(_bits(got), _bits(oracle.gemm(a, b, 14, int(mode))))


@pytest.mark.parametrize("lda_pad,ldb_pad", [(1, 0), (0, 1), (2, 3), (8, 8)])
def test_fused_k1_leading_dimensions(ctx, oracle, lda_pad, ldb_pad):
    """odd leading dimensions take the two-kernel rows path, even ones the fused one"""
    m, n, k = 190, 77, 1500
    a = gen_matrix(m, k, 0.5, 21)
    b = gen_matrix(k, n, 0.5, 22)
    got = _run(ctx, a, b, EmuConfig(n_moduli=16), lda=m + lda_pad, ldb=k + ldb_pad)
    np.testing.assert_array_equal(_bits(got), _bits(oracle.gemm(a, b, 16, 0)))


@pytest.mark.parametrize("N,mode", [(8, ScaleMode.Fast), (10, ScaleMode.Accurate), (6, ScaleMode.Fast)])
def test_fused_k1_fp32(ctx, oracle, N, mode):
    m, n, k = 321, 190, 2500
    a = gen_matrix(m, k, 0.5, 31).astype(np.float32)
    b = gen_matrix(k, n, 0.5, 32).astype(np.float32)
    cfg = EmuConfig(n_moduli=N, mode=mode, precision=Precision.Fp32)
    A, B = _dev(a), _dev(b)
    C = _dev(np.zeros((m, n)))
    ctx.gemm(A, B, cfg, C)
    want = oracle.gemm(a, b, N, int(mode), prec=1)
    np.testing.assert_array_equal(_bits(C.cpu().numpy()), _bits(want))


@pytest.mark.parametrize("ta,tb", [(False, False), (True, True)])
def test_fused_k1_flagged_lines(ctx, oracle, ta, tb):
    """rows / columns whose maxima leave the a^2-safe range take the exact
    sequential recompute inside the fused finalize (row groups: the last slice's
    block; columns: warp 0 of the column's block)"""
    m, n, k = 190, 130, 3000
    a = gen_matrix(m, k, 0.5, 41)
    b = gen_matrix(k, n, 0.5, 42)
    a[[3, 70, m - 1], :] *= 2.0 ** -450
    a[[9, 100], :] *= 2.0 ** 510
    b[:, [0, 64, n - 1]] *= 2.0 ** -450
    b[:, [11]] *= 2.0 ** 505
    got = _run(ctx, a, b, EmuConfig(n_moduli=14), ta, tb)
    np.testing.assert_array_equal(_bits(got), _bits(oracle.gemm(a, b, 14, 0)))


def test_fused_k1_state_across_calls(ctx, oracle):
    """the ticket counters, row accumulators, group counters and group flags
    reset themselves at the end of each launch — so many calls of changing
    shapes on one handle (both K1 streams) stay exact"""
    rng = np.random.default_rng(5)
    for it in range(24):
        m, n, k = (int(v) for v in rng.integers(1, 700, size=3))
        mode = ScaleMode(int(rng.integers(0, 2)))
        ta, tb = bool(rng.integers(0, 2)), bool(rng.integers(0, 2))
        a = gen_matrix(m, k, 1.0, 100 + it)
        b = gen_matrix(k, n, 1.0, 200 + it)
        got = _run(ctx, a, b, EmuConfig(n_moduli=13, mode=mode), ta, tb)
        np.testing.assert_array_equal(_bits(got), _bits(oracle.gemm(a, b, 13, int(mode))),
                                      err_msg=f"call {it}: {m}x{n}x{k} {mode.name} ta={ta} tb={tb}")


@pytest.mark.parametrize("where", ["a_row", "b_col"])
@pytest.mark.parametrize("bad", [np.inf, np.nan])
@pytest.mark.parametrize("trans", [False, True])
def test_fused_k1_nonfinite(ctx, where, bad, trans):
    m, n, k = 150, 90, 700
    a = gen_matrix(m, k, 0.5, 51)
    b = gen_matrix(k, n, 0.5, 52)
    if where == "a_row":
        a[77, 300] = bad
    else:
        b[650, 45] = bad
    with pytest.raises(InputError):
        _run(ctx, a, b, EmuConfig(n_moduli=14), trans, trans)
    # the handle is still usable afterwards (state reset by the failing call's kernels)
    a2 = gen_matrix(m, k, 0.5, 53)
    b2 = gen_matrix(k, n, 0.5, 54)
    _run(ctx, a2, b2, EmuConfig(n_moduli=14), trans, trans)


@pytest.mark.parametrize("mode", [ScaleMode.Fast, ScaleMode.Accurate])
def test_fused_k1_cuda_graph_replay(oracle, mode):
    """a captured call replays on new inputs: the one-pass kernels bake no
    per-call state into the graph (run again with the row kernel on below)"""
    from paper_2508_03984_b200 import Context

    m, n, k = 640, 384, 1100
    ctx = Context(0)
    cfg = EmuConfig(n_moduli=14, mode=mode, stream_ordered=True)
    a0, b0 = gen_matrix(m, k, 0.5, 1), gen_matrix(k, n, 0.5, 2)
    a1, b1 = gen_matrix(m, k, 1.0, 3), gen_matrix(k, n, 1.0, 4)
    A, B, C = _dev(a0), _dev(b0), _dev(np.zeros((m, n)))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ctx.set_stream(s.cuda_stream)
        ctx.gemm(A, B, cfg, C)  # warm-up: sizes the workspace and clears the state
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            ctx.set_stream(torch.cuda.current_stream().cuda_stream)
            ctx.gemm(A, B, cfg, C)
    for a, b in ((a1, b1), (a0, b0), (a1, b1)):
        A.copy_(_dev(a))
        B.copy_(_dev(b))
        g.replay()
        torch.cuda.synchronize()
        np.testing.assert_array_equal(_bits(C.cpu().numpy()), _bits(oracle.gemm(a, b, 14, int(mode))))
    ctx.close()


@pytest.mark.parametrize("mask", ["1", "3"])
def test_row_kernel_enabled_subprocess(mask):
    """This module again with the one-pass kernels taken at every size
    (OZK_K1_FUSED_ANY: by default the column kernel serves only columns of
    >= 4096 elements, >= 1024 of them): mask 1 the column kernel, mask 3 also
    the opt-in row kernel."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, OZK_K1_FUSED=mask, OZK_K1_FUSED_ANY="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", __file__,
                        "-k", "not subprocess"], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("lag", ["1", "100000"])
def test_fused_k1_row_lag_extremes(ctx, oracle, lag, monkeypatch):
    """the row kernel's statistics/planes distance at its floor (one group of
    slices: the deadlock-freedom bound) and unbounded; read per launch"""
    monkeypatch.setenv("OZK_K1_LAG", lag)
    for m, n, k in [(700, 90, 5000), (2049, 64, 1000)]:
        a = gen_matrix(m, k, 1.0, 61 + m)
        b = gen_matrix(k, n, 1.0, 62 + n)
        got = _run(ctx, a, b, EmuConfig(n_moduli=14))
        np.testing.assert_array_equal(_bits(got), _bits(oracle.gemm(a, b, 14, 0)))


@pytest.mark.parametrize("ta,tb", [(False, False), (True, True)])
def test_fused_k1_subnormal_lines(ctx, oracle, ta, tb):
    """The line maxima are taken on the high words of the bit patterns
    (k1_line.cuh AbsMax): lines of subnormals whose high words are all zero
    (|x| < 2^-1042) must still count as nonzero and take the exact recompute,
    lines of larger subnormals keep their exponent; the scale exponents and C
    must match the reference."""
    m, n, k = 130, 70, 900
    a = gen_matrix(m, k, 0.5, 91)
    b = gen_matrix(k, n, 0.5, 92)
    a[5, :] = np.ldexp(a[5, :], -1062)     # high words 0: only the low words are nonzero
    a[6, :] = np.ldexp(a[6, :], -1030)     # subnormal, high words nonzero
    a[7, :] = 0.0
    a[7, 3] = np.ldexp(1.0, -1070)          # a single tiny element in a zero row
    b[:, 9] = np.ldexp(b[:, 9], -1062)
    b[:, 10] = np.ldexp(b[:, 10], -1026)
    b[:, 11] = 0.0
    b[400, 11] = -np.ldexp(1.0, -1073)
    wmu, wnu = oracle.scale(a, b, 14, 0)
    mu = torch.zeros(m, dtype=torch.int32, device="cuda")
    nu = torch.zeros(n, dtype=torch.int32, device="cuda")
    ctx.stage_scale(_dev(a), _dev(b), EmuConfig(n_moduli=14), mu, nu)
    np.testing.assert_array_equal(mu.cpu().numpy(), wmu)
    np.testing.assert_array_equal(nu.cpu().numpy(), wnu)
    for mode in (ScaleMode.Fast, ScaleMode.Accurate):
        got = _run(ctx, a, b, EmuConfig(n_moduli=14, mode=mode), ta, tb)
        np.testing.assert_array_equal(_bits(got), _bits(oracle.gemm(a, b, 14, int(mode))))
