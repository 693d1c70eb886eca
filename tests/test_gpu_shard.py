"""The column-shard API (ozk_shard_begin / _rowmax / _end) on the GPU.

One B200 stands in for W ranks: W handles each take a contiguous column block
of B, the accurate-mode partial row maxima are max-reduced exactly as
distributed.gemm_sharded's all-reduce would, and the concatenated shards must
equal the single-call result bit for bit (which the oracle pins). The NCCL
exchange itself is covered with gloo in tests/test_distributed.py.
"""
import numpy as np
import pytest

from paper_2508_03984_b200 import Context, EmuConfig, ScaleMode, gen_matrix
from paper_2508_03984_b200.distributed import column_shard

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
