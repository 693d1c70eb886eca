"""Bounded workspace: problems larger than the handle's workspace limit run in
row x column panels (api.cu make_plan / run_panels). Every stage after the
O(m + n) exponents is row/column-local, so a panelled call must equal the
one-panel call bit for bit (which the oracle pins, tests/test_gpu_parity.py);
tiny limits force many panels, both loop orders, partial edge panels, every
operand layout, accurate mode, FP32 tables, alpha/beta and k > 2^17.
"""
import numpy as np
import pytest

from paper_2508_03984_b200 import Context, EmuConfig, Precision, ScaleMode, gen_matrix

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t()


def _bits(x):
    x = np.ascontiguousarray(x)
    return x.view(np.int64 if x.dtype == np.float64 else np.int32)


def _ws(N, m, n, k, mr, nc):
    """workspace of one (mr x nc) panel: A planes + B planes + U (untransposed)"""
    ld = lambda x: (x + 15) // 16 * 16  # noqa: E731
    return N * (k * ld(mr) + nc * ld(k) + nc * ld(mr))


@pytest.fixture(scope="module")
def big():
    return Context(0)


@pytest.fixture(scope="module")
def small():
    return Context(0)


def _pair(big, small, A, B, cfg, limit, alpha=1.0, beta=0.0, C0=None, ta=False, tb=False, c32=False):
    m = A.shape[1] if ta else A.shape[0]
    n = B.shape[0] if tb else B.shape[1]
    dt = torch.float32 if c32 else torch.float64
    outs = []
    for ctx, lim in ((big, 0), (small, limit)):
        ctx.set_workspace_limit(lim)
        C = torch.zeros((n, m), dtype=dt, device="cuda").t()
        if C0 is not None:
            C.copy_(C0)
        ctx.gemm(A, B, cfg, C, alpha=alpha, beta=beta, trans_a=ta, trans_b=tb)
        torch.cuda.synchronize()
        outs.append(C.cpu().numpy())
    return outs, big.last_plan, small.last_plan


@pytest.mark.parametrize("mode", [ScaleMode.Fast, ScaleMode.Accurate])
@pytest.mark.parametrize("m,n", [(1500, 700), (700, 1500)])
def test_panels_equal_single(big, small, mode, m, n):
    """(1500, 700): column panels outside (A re-derived per column panel);
    (700, 1500): row panels outside"""
    k = 300
    N = 14
    a, b = gen_matrix(m, k, 1.0, 91), gen_matrix(k, n, 1.0, 92)
    b[:, 3] = 0.0
    lim = _ws(N, m, n, k, 256, 256) + 1024
    (one, many), p1, p2 = _pair(big, small, _dev(a), _dev(b), EmuConfig(n_moduli=N, mode=mode), lim)
    assert p1["panels"] == 1 and p2["panels"] == ((m + 255) // 256) * ((n + 255) // 256)
    assert p2["extra_passes"] == (min(m, n) + 255) // 256 - 1
    np.testing.assert_array_equal(_bits(many), _bits(one))


@pytest.mark.parametrize("ta,tb", [(True, False), (False, True), (True, True)])
def test_panels_transposed(big, small, ta, tb):
    m, n, k = 900, 600, 280
    a, b = gen_matrix(m, k, 0.5, 93), gen_matrix(k, n, 0.5, 94)
    A = _dev(np.asfortranarray(a.T)) if ta else _dev(a)
    B = _dev(np.asfortranarray(b.T)) if tb else _dev(b)
    lim = 3 * _ws(14, m, n, k, 256, 256)
    (one, many), _, p2 = _pair(big, small, A, B, EmuConfig(n_moduli=14), lim, ta=ta, tb=tb)
    assert p2["panels"] > 1
    np.testing.assert_array_equal(_bits(many), _bits(one))


def test_panels_alpha_beta_fp32(big, small):
    m, n, k = 800, 560, 333
    a, b = gen_matrix(m, k, 0.5, 95), gen_matrix(k, n, 0.5, 96)
    c0 = torch.from_numpy(np.ascontiguousarray(gen_matrix(m, n, 0.0, 97).T)).cuda().t()
    lim = 2 * _ws(14, m, n, k, 256, 256)
    (one, many), _, p2 = _pair(big, small, _dev(a), _dev(b), EmuConfig(n_moduli=14), lim, alpha=-0.75, beta=1.25,
                               C0=c0)
    assert p2["panels"] > 1
    np.testing.assert_array_equal(_bits(many), _bits(one))
    # FP32 tables with FP32 inputs and an FP32 C
    a32, b32 = a.astype(np.float32), b.astype(np.float32)
    cfg = EmuConfig(n_moduli=8, mode=ScaleMode.Accurate, precision=Precision.Fp32)
    (one, many), _, p2 = _pair(big, small, _dev(a32), _dev(b32), cfg, lim // 2, c32=True)
    assert p2["panels"] > 1
    np.testing.assert_array_equal(_bits(many), _bits(one))


def test_panels_long_k(big, small, oracle):
    """k > 2^17: each panel's K2 runs in 2^17 chunks with the mod-accumulate epilogue"""
    m, n, k = 300, 280, (1 << 17) + 40
    a, b = gen_matrix(m, k, 0.5, 98), gen_matrix(k, n, 0.5, 99)
    lim = _ws(12, m, n, k, 256, 256) + 4096
    (one, many), _, p2 = _pair(big, small, _dev(a), _dev(b), EmuConfig(n_moduli=12), lim)
    assert p2["panels"] == 4
    np.testing.assert_array_equal(_bits(many), _bits(one))
    np.testing.assert_array_equal(_bits(one), _bits(oracle.gemm(a, b, 12, 0)))


def test_panels_host_call(small, oracle):
    """ozk_gemm_host beyond the limit: whole operands to the device, panelled call, C back"""
    m, n, k = 600, 520, 200
    a, b = gen_matrix(m, k, 0.5, 100), gen_matrix(k, n, 0.5, 101)
    small.set_workspace_limit(_ws(14, m, n, k, 256, 256) + 1024)
    for mode in (ScaleMode.Fast, ScaleMode.Accurate):
        got = small.gemm_host(a, b, EmuConfig(n_moduli=14, mode=mode))
        assert small.last_plan["panels"] == 9
        np.testing.assert_array_equal(_bits(got), _bits(oracle.gemm(a, b, 14, int(mode))))
    small.set_workspace_limit(0)


def test_workspace_is_bounded(small):
    """a limit caps what the handle holds for the planes and U"""
    m, n, k = 2048, 2048, 1024
    a, b = gen_matrix(m, k, 0.5, 102), gen_matrix(k, n, 0.5, 103)
    fresh = Context(0)
    lim = 40 << 20
    fresh.set_workspace_limit(lim)
    C = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
    fresh.gemm(_dev(a), _dev(b), EmuConfig(n_moduli=14), C)
    torch.cuda.synchronize()
    assert fresh.last_plan["panels"] > 1
    assert fresh.workspace_bytes < lim + (8 << 20)  # + the O(m + n) exponent/statistics buffers
    fresh.close()
