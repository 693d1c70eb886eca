"""Stream-ordered calls (OZK_FLAG_ASYNC / EmuConfig.stream_ordered): no host
sync per call, the deferred non-finite check, and CUDA-graph capture of a
whole emulated GEMM — all bit-identical to the synchronous call."""
import numpy as np
import pytest

from paper_2508_03984_b200 import Context, EmuConfig, ScaleMode, gen_matrix
from paper_2508_03984_b200.emulator import InputError

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t()


def _bits(x):
    return np.ascontiguousarray(x).view(np.int64)


@pytest.mark.parametrize("mode", [ScaleMode.Fast, ScaleMode.Accurate])
def test_stream_ordered_equals_sync(oracle, mode):
    m, n, k = 300, 200, 700
    a, b = gen_matrix(m, k, 0.5, 61), gen_matrix(k, n, 0.5, 62)
    ctx = Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    cfg = EmuConfig(n_moduli=14, mode=mode, stream_ordered=True)
    outs = []
    for _ in range(3):  # back to back, one sync at the end
        C = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
        ctx.gemm(_dev(a), _dev(b), cfg, C)
        outs.append(C)
    ctx.synchronize()
    want = oracle.gemm(a, b, 14, int(mode))
    for C in outs:
        np.testing.assert_array_equal(_bits(C.cpu().numpy()), _bits(want))


def test_deferred_nonfinite_check():
    m = n = k = 64
    a, b = gen_matrix(m, k, 0.5, 1), gen_matrix(k, n, 0.5, 2)
    a[5, 7] = np.nan
    ctx = Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    C = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
    ctx.gemm(_dev(a), _dev(b), EmuConfig(n_moduli=14, stream_ordered=True), C)  # no raise here
    a[5, 7] = 1.0
    ctx.gemm(_dev(a), _dev(b), EmuConfig(n_moduli=14, stream_ordered=True), C)  # a clean call does not clear it
    with pytest.raises(InputError):
        ctx.synchronize()
    ctx.synchronize()  # collected and cleared
    with pytest.raises(InputError):  # the synchronous call still raises at once
        a[0, 0] = np.inf
        ctx.gemm(_dev(a), _dev(b), EmuConfig(n_moduli=14), C)


@pytest.mark.parametrize("m,n,k,mode", [(1024, 1024, 1024, ScaleMode.Accurate), (700, 513, 300, ScaleMode.Fast)])
def test_cuda_graph_capture(oracle, m, n, k, mode):
    """warm up (sizes the workspace), capture one call, replay it on new inputs"""
    a0, b0 = gen_matrix(m, k, 0.5, 71), gen_matrix(k, n, 0.5, 72)
    a1, b1 = gen_matrix(m, k, 1.0, 73), gen_matrix(k, n, 1.0, 74)
    A, B = _dev(a0), _dev(b0)
    C = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
    ctx = Context(0)
    cfg = EmuConfig(n_moduli=14, mode=mode, stream_ordered=True)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        ctx.set_stream(side.cuda_stream)
        ctx.gemm(A, B, cfg, C)
        ctx.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ctx.set_stream(torch.cuda.current_stream().cuda_stream)
        ctx.gemm(A, B, cfg, C)
    A.copy_(_dev(a1))
    B.copy_(_dev(b1))
    g.replay()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(_bits(C.cpu().numpy()), _bits(oracle.gemm(a1, b1, 14, int(mode))))
    A.copy_(_dev(a0))
    B.copy_(_dev(b0))
    g.replay()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(_bits(C.cpu().numpy()), _bits(oracle.gemm(a0, b0, 14, int(mode))))
