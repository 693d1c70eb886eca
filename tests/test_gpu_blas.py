"""GPU parity of the BLAS front end: transposed operands,
leading dimensions larger than the matrix, alpha/beta, strided batches.

The reference takes op(X) = X only (emulator.hpp:23-32), so every case is
checked against the oracle run on the explicitly transposed operands:
gemm(op(A), op(B)) must match bit for bit, whichever way A and B are stored.
"""
import numpy as np
import pytest

from paper_2508_03984_b200 import ConfigError, EmuConfig, InputError, Precision, ScaleMode, gen_matrix
from paper_2508_03984_b200 import _lib

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _bits(x):
    return np.ascontiguousarray(x).view(np.int64 if x.dtype == np.float64 else np.int32)


def _dev(x: np.ndarray, ld: int | None = None, dtype=None):
    """host matrix -> column-major CUDA tensor view with leading dimension ld"""
    rows, cols = x.shape
    ld = rows if ld is None else ld
    buf = np.full((cols, ld), np.nan, dtype=dtype or x.dtype)  # padding rows are NaN: must never be read
    buf[:, :rows] = x.T
    return torch.from_numpy(buf).cuda().t()[:rows]


def _stored(op: np.ndarray, trans: bool) -> np.ndarray:
    return np.asfortranarray(op.T) if trans else np.asfortranarray(op)


TRANS = [(False, False), (True, False), (False, True), (True, True)]
CASES = [(1, 1, 1), (33, 65, 127), (256, 256, 256), (300, 129, 1000), (129, 520, 77), (600, 700, 300)]


@pytest.mark.parametrize("ta,tb", TRANS)
@pytest.mark.parametrize("m,n,k", CASES)
@pytest.mark.parametrize("mode", [ScaleMode.Fast, ScaleMode.Accurate])
def test_transposes_fp64(ctx, oracle, ta, tb, m, n, k, mode):
    a = gen_matrix(m, k, 1.0, 71)
    b = gen_matrix(k, n, 1.0, 72)
    A, B = _dev(_stored(a, ta)), _dev(_stored(b, tb))
    Cg = _dev(np.zeros((m, n)))
    ctx.gemm(A, B, EmuConfig(n_moduli=14, mode=mode), Cg, trans_a=ta, trans_b=tb)
    want = oracle.gemm(a, b, 14, int(mode))
    np.testing.assert_array_equal(_bits(Cg.cpu().numpy()), _bits(want))


@pytest.mark.parametrize("ta,tb", TRANS)
@pytest.mark.parametrize("mode", [ScaleMode.Fast, ScaleMode.Accurate])
@pytest.mark.parametrize("f32_inputs", [True, False])
def test_transposes_fp32(ctx, oracle, ta, tb, mode, f32_inputs):
    m, n, k = 200, 150, 700
    a = gen_matrix(m, k, 1.0, 73)
    b = gen_matrix(k, n, 1.0, 74)
    dt = np.float32 if f32_inputs else np.float64
    A, B = _dev(_stored(a, ta).astype(dt)), _dev(_stored(b, tb).astype(dt))
    Cg = _dev(np.zeros((m, n)))  # the reference returns FP64 C for FP32 emulation too
    ctx.gemm(A, B, EmuConfig(n_moduli=8, mode=mode, precision=Precision.Fp32), Cg, trans_a=ta, trans_b=tb)
    want = oracle.gemm(a.astype(np.float32), b.astype(np.float32), 8, int(mode), prec=1)
    np.testing.assert_array_equal(_bits(Cg.cpu().numpy()), _bits(want))


@pytest.mark.parametrize("ta,tb", TRANS)
def test_leading_dimensions_and_alpha_beta(ctx, oracle, ta, tb):
    """lda/ldb/ldc larger than the rows (NaN padding must never be read)"""
    m, n, k = 70, 90, 130
    a = gen_matrix(m, k, 0.5, 75)
    b = gen_matrix(k, n, 0.5, 76)
    c0 = gen_matrix(m, n, 0.5, 77)
    sa, sb = _stored(a, ta), _stored(b, tb)
    A, B = _dev(sa, ld=sa.shape[0] + 13), _dev(sb, ld=sb.shape[0] + 5)
    Cg = _dev(c0, ld=m + 3)
    ctx.gemm(A, B, EmuConfig(n_moduli=13), Cg, alpha=0.5, beta=-2.0, trans_a=ta, trans_b=tb)
    want = 0.5 * oracle.gemm(a, b, 13, 0) + (-2.0) * c0
    np.testing.assert_array_equal(_bits(Cg.cpu().numpy()), _bits(want))


@pytest.mark.parametrize("ta,tb", TRANS)
@pytest.mark.parametrize("mode", [ScaleMode.Fast, ScaleMode.Accurate])
def test_transposes_host_multiblock(ctx, oracle, ta, tb, mode):
    """ozk_gemm_host with column blocks: trans_b blocks are pitched row ranges"""
    m, n, k = 260, 2600, 333
    a = gen_matrix(m, k, 1.0, 78)
    b = gen_matrix(k, n, 1.0, 79)
    got = ctx.gemm_host(_stored(a, ta), _stored(b, tb), EmuConfig(n_moduli=14, mode=mode), trans_a=ta, trans_b=tb)
    np.testing.assert_array_equal(_bits(got), _bits(oracle.gemm(a, b, 14, int(mode))))


@pytest.mark.parametrize("ta,tb", [(True, False), (False, True)])
def test_transposes_long_k(ctx, oracle, ta, tb):
    """k > 2^17 runs K2 in chunks; the chunk offset differs per operand major"""
    m, n, k = 9, 7, (1 << 17) + 1000
    a = gen_matrix(m, k, 0.5, 80)
    b = gen_matrix(k, n, 0.5, 81)
    Cg = _dev(np.zeros((m, n)))
    ctx.gemm(_dev(_stored(a, ta)), _dev(_stored(b, tb)), EmuConfig(n_moduli=14), Cg, trans_a=ta, trans_b=tb)
    np.testing.assert_array_equal(_bits(Cg.cpu().numpy()), _bits(oracle.gemm(a, b, 14, 0)))


def test_dgemm_ex_chars(ctx, oracle):
    m, n, k = 40, 50, 60
    a = gen_matrix(m, k, 0.5, 82)
    b = gen_matrix(k, n, 0.5, 83)
    A, B = _dev(_stored(a, True)), _dev(_stored(b, True))
    Cg = _dev(np.zeros((m, n)))
    L = _lib.load()
    _lib.check(L.ozk_dgemm_ex(ctx.handle, 14, 0, b"T", b"t", m, n, k, 1.0, A.data_ptr(), k, B.data_ptr(), n, 0.0,
                              Cg.data_ptr(), m))
    np.testing.assert_array_equal(_bits(Cg.cpu().numpy()), _bits(oracle.gemm(a, b, 14, 0)))
    with pytest.raises(ConfigError):
        _lib.check(L.ozk_dgemm_ex(ctx.handle, 14, 0, b"X", b"N", m, n, k, 1.0, A.data_ptr(), k, B.data_ptr(), n,
                                  0.0, Cg.data_ptr(), m))


def test_transposed_leading_dimension_checked(ctx):
    """lda >= k for trans_a, ldb >= n for trans_b (validate order as gemm_emulated)"""
    A = _dev(np.zeros((5, 7)))  # stored 5 x 7 -> op(A) 7 x 5 with lda 5 = k: fine
    B = _dev(np.zeros((3, 5)))  # stored 3 x 5 -> op(B) 5 x 3 with ldb 3 = n: fine
    Cg = _dev(np.zeros((7, 3)))
    ctx.gemm(A, B, EmuConfig(n_moduli=8), Cg, trans_a=True, trans_b=True)
    L = _lib.load()
    conf = _lib.OzkConfig()
    conf.n_moduli, conf.block_k, conf.flags = 8, 1 << 17, _lib.OZK_FLAG_TRANS_A
    import ctypes as C

    with pytest.raises(InputError):  # lda 4 < k 5
        _lib.check(L.ozk_gemm(ctx.handle, C.byref(conf), 7, 3, 5, 1.0, A.data_ptr(), 4, B.data_ptr(), 5, 0.0,
                              Cg.data_ptr(), 7))


@pytest.mark.parametrize("ta,tb", [(False, False), (True, True)])
def test_strided_batched(ctx, oracle, ta, tb):
    batch, m, n, k = 3, 50, 40, 70
    As = [gen_matrix(m, k, 0.5, 90 + i) for i in range(batch)]
    Bs = [gen_matrix(k, n, 0.5, 95 + i) for i in range(batch)]

    def stack(mats, trans):
        st = [_stored(x, trans) for x in mats]
        r, c = st[0].shape
        buf = np.stack([x.T for x in st])  # (batch, cols, rows) row-major == column-major slices
        return torch.from_numpy(np.ascontiguousarray(buf)).cuda().transpose(1, 2)

    A, B = stack(As, ta), stack(Bs, tb)
    Cg = torch.zeros((batch, n, m), dtype=torch.float64, device="cuda").transpose(1, 2)
    ctx.gemm_strided_batched(A, B, EmuConfig(n_moduli=12), Cg, trans_a=ta, trans_b=tb)
    got = Cg.cpu().numpy()
    for i in range(batch):
        np.testing.assert_array_equal(_bits(got[i]), _bits(oracle.gemm(As[i], Bs[i], 12, 0)))
