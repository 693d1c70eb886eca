"""The column-shard API (ozk_shard_begin / _rowmax / _end) and the
row-streamed shard (ozk_shard_stream_begin / _rows / _end) on the GPU.

One B200 stands in for W ranks: W handles each take a contiguous column block
of B, the accurate-mode partial row maxima are max-reduced exactly as
distributed.gemm_sharded's all-reduce would, and the concatenated shards must
equal the single-call result bit for bit (which the oracle pins). The NCCL
exchange itself is covered with gloo in tests/test_distributed.py.
"""
import numpy as np
import pytest

from paper_2508_03984_b200 import Context, EmuConfig, Precision, ScaleMode, gen_matrix
from paper_2508_03984_b200.distributed import column_shard, row_blocks
from paper_2508_03984_b200.emulator import ConfigError, InputError

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t()


def _bits(x):
    return np.ascontiguousarray(x).view(np.int64)


def _sharded(ctxs, A, B, cfg):
    m, n = A.shape[0], B.shape[1]
    W = len(ctxs)
    blocks = [column_shard(n, W, r) for r in range(W)]
    outs = []
    for ctx, (j0, nj) in zip(ctxs, blocks):
        ctx.shard_begin(A, B[:, j0:j0 + nj], cfg)
    if cfg.mode == ScaleMode.Accurate:  # the all-reduce(MAX) of gemm_sharded
        rms = [ctx.shard_rowmax() for ctx in ctxs]
        red = torch.stack(rms).amax(dim=0)
        for r in rms:
            r.copy_(red)
    for ctx, (j0, nj) in zip(ctxs, blocks):
        C = torch.zeros((nj, m), dtype=torch.float64, device="cuda").t()
        ctx.shard_end(C)
        outs.append(C)
    torch.cuda.synchronize()
    return torch.cat(outs, dim=1).cpu().numpy()


@pytest.mark.parametrize("mode", [ScaleMode.Fast, ScaleMode.Accurate])
@pytest.mark.parametrize("W", [2, 3, 8])
def test_shards_concatenate_to_oracle(oracle, mode, W):
    m, n, k = 150, 301, 400
    a = gen_matrix(m, k, 2.0, 31)
    b = gen_matrix(k, n, 2.0, 32)
    b[:, 5] = 0.0  # a zero column inside the first shard
    ctxs = [Context(0) for _ in range(W)]
    got = _sharded(ctxs, _dev(a), _dev(b), EmuConfig(n_moduli=14, mode=mode))
    np.testing.assert_array_equal(_bits(got), _bits(oracle.gemm(a, b, 14, int(mode))))


@pytest.mark.parametrize("mode", [ScaleMode.Fast, ScaleMode.Accurate])
def test_shards_full_size(mode):
    """n = 16384 split over 8 shards (the bench's per-rank layout) == one call"""
    n = 16384
    g = torch.Generator(device="cuda").manual_seed(5)
    A = ((torch.rand((n, n), generator=g, device="cuda", dtype=torch.float64) - 0.5)
         * torch.exp(0.5 * torch.randn((n, n), generator=g, device="cuda", dtype=torch.float64))).t()
    B = ((torch.rand((n, n), generator=g, device="cuda", dtype=torch.float64) - 0.5)
         * torch.exp(0.5 * torch.randn((n, n), generator=g, device="cuda", dtype=torch.float64))).t()
    cfg = EmuConfig(n_moduli=14, mode=mode)
    ctx = Context(0)
    C = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
    ctx.gemm(A, B, cfg, C)
    want = C.cpu().numpy()
    del C
    got = _sharded([Context(0) for _ in range(8)], A, B, cfg)
    np.testing.assert_array_equal(_bits(got), _bits(want))


def _streamed(ctx, A, B, cfg, C, row_block, alpha=1.0, beta=0.0, packed=False):
    """A fed to ozk_shard_stream_rows block by block, either as views into A
    (lda = m) or as packed mr x k copies (what a broadcast delivers)"""
    m, k = A.shape
    ctx.shard_stream_begin(m, k, B, cfg, C, alpha, beta)
    for r0, mr in row_blocks(m, row_block):
        rows = A[r0:r0 + mr]
        if packed:
            p = torch.empty((k, mr), dtype=A.dtype, device=A.device).t()
            p.copy_(rows)
            rows = p
        ctx.shard_stream_rows(r0, rows)
    ctx.shard_stream_end()


@pytest.mark.parametrize("packed", [False, True])
@pytest.mark.parametrize("m,n,k,N,phi,rb", [(1000, 300, 700, 14, 0.5, 128), (257, 129, 1000, 12, 2.0, 100),
                                             (33, 500, 4000, 20, 1.0, 8)])
def test_stream_rows_equal_single_call(oracle, packed, m, n, k, N, phi, rb):
    a = gen_matrix(m, k, phi, 41)
    b = gen_matrix(k, n, phi, 42)
    a[3, :] = 0.0  # a zero row in the first block
    cfg = EmuConfig(n_moduli=N, mode=ScaleMode.Fast)
    ctx = Context(0)
    C = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
    _streamed(ctx, _dev(a), _dev(b), cfg, C, rb, packed=packed)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(_bits(C.cpu().numpy()), _bits(oracle.gemm(a, b, N, 0)))


def test_stream_rows_alpha_beta_and_fp32():
    m, n, k = 700, 260, 900
    a = gen_matrix(m, k, 0.5, 43)
    b = gen_matrix(k, n, 0.5, 44)
    c0 = gen_matrix(m, n, 0.5, 45)
    ctx = Context(0)
    cfg = EmuConfig(n_moduli=14, mode=ScaleMode.Fast)
    want = _dev(c0)
    ctx.gemm(_dev(a), _dev(b), cfg, want, alpha=-0.75, beta=1.5)
    got = _dev(c0)
    _streamed(ctx, _dev(a), _dev(b), cfg, got, 256, alpha=-0.75, beta=1.5)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(_bits(got.cpu().numpy()), _bits(want.cpu().numpy()))
    # FP32 operands at FP32 precision, FP32 C
    a32 = _dev(a.astype(np.float32))
    b32 = _dev(b.astype(np.float32))
    cfg32 = EmuConfig(n_moduli=8, mode=ScaleMode.Fast, precision=Precision.Fp32)
    want32 = torch.zeros((n, m), dtype=torch.float32, device="cuda").t()
    ctx.gemm(a32, b32, cfg32, want32)
    got32 = torch.zeros((n, m), dtype=torch.float32, device="cuda").t()
    _streamed(ctx, a32, b32, cfg32, got32, 200)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got32.cpu().numpy().view(np.int32), want32.cpu().numpy().view(np.int32))


def test_stream_rows_errors():
    m, n, k = 64, 64, 64
    A = _dev(gen_matrix(m, k, 0.5, 1))
    B = _dev(gen_matrix(k, n, 0.5, 2))
    C = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
    ctx = Context(0)
    with pytest.raises(ConfigError):  # accurate-mode mu needs every column first
        ctx.shard_stream_begin(m, k, B, EmuConfig(n_moduli=14, mode=ScaleMode.Accurate), C)
    with pytest.raises(InputError):
        ctx.shard_stream_rows(0, A)  # no open stream
    ctx.shard_stream_begin(m, k, B, EmuConfig(n_moduli=14), C)
    with pytest.raises(InputError):
        ctx.shard_stream_rows(48, A[0:32])  # past row m
    with pytest.raises(InputError):
        ctx.shard_stream_rows(8, A[0:8])  # r0 not a multiple of 16
    ctx.shard_stream_rows(0, A[0:32])
    with pytest.raises(InputError):
        ctx.shard_stream_end()  # rows 32..63 never arrived


def test_stream_rows_full_size():
    """16384^3 N = 14 fast, streamed in packed 2048-row blocks (the bench's
    multi-GPU path) == one call, bit for bit"""
    n = 16384
    g = torch.Generator(device="cuda").manual_seed(6)
    A = ((torch.rand((n, n), generator=g, device="cuda", dtype=torch.float64) - 0.5)
         * torch.exp(0.5 * torch.randn((n, n), generator=g, device="cuda", dtype=torch.float64))).t()
    B = ((torch.rand((n, n), generator=g, device="cuda", dtype=torch.float64) - 0.5)
         * torch.exp(0.5 * torch.randn((n, n), generator=g, device="cuda", dtype=torch.float64))).t()
    cfg = EmuConfig(n_moduli=14, mode=ScaleMode.Fast)
    ctx = Context(0)
    C = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
    ctx.gemm(A, B, cfg, C)
    want = C.cpu().numpy()
    _streamed(ctx, A, B, cfg, C, 2048, packed=True)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(_bits(C.cpu().numpy()), _bits(want))
