"""K3 variants held to the production bar. The default K3 for FP64 tables
(csrc/k3_tc.cu) takes C1 and an interval for C2 from one u8 x u8 tcgen05 MMA
and replays the reference's sequential C2 only where the interval cannot
decide the final rounding; the all-FP64 kernel (csrc/k3_reconstruct.cu) takes
FP32 tables and OZK_K3_TC=0. The library reads both switches once per process,
so the sweeps run in child processes:
  * OZK_K3_REPLAY_ALL=1 widens the interval so (almost) every element takes the
    replay path — the path the default run reaches only ~100 times per 16384^2;
  * OZK_K3_TC=0 runs every FP64 case through the all-FP64 kernel;
  * OZK_K3_CW=8 runs the column-tiled kernel with 8 consumer warps, and
    OZK_K3_TILE=1 the earlier 512-row x 1-column kernel."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{"OZK_K3_REPLAY_ALL": "1"}, {"OZK_K3_TC": "0"},
                                 {"OZK_K3_CW": "8", "OZK_K3_REPLAY_ALL": "1"}, {"OZK_K3_TILE": "1"},
                                 {"OZK_K3_FULL": "0"}, {"OZK_K3_TILE": "8"}, {"OZK_K3_TILE": "8", "OZK_K3_REPLAY_ALL": "1"}],
                         ids=["replay_all", "fp64_kernel", "cw8_replay_all", "row_tile_kernel", "no_full_tiles",
                              "tile8", "tile8_replay_all"])
def test_k3_variant_random_sweep(env):
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_random.py"), os.path.join(ROOT, "tests", "test_gpu_parity.py"),
                        os.path.join(ROOT, "tests", "test_gpu_k3_tc.py") + "::test_k3_full_tiles"],
                       cwd=ROOT, env=dict(os.environ, **env), capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


def test_k3_replays_are_rare_and_exact(oracle):
    """N = 14 at a size where the interval fails for a handful of elements:
    the count is small and the result still equals the oracle bit for bit."""
    torch = pytest.importorskip("torch")
    from paper_2508_03984_b200 import Context, EmuConfig, gen_matrix

    ctx = Context(0)
    m, n, k = 1024, 1024, 512
    a = gen_matrix(m, k, 0.5, 11)
    b = gen_matrix(k, n, 0.5, 12)
    ctx.k3_replays(reset=True)
    A = torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()
    B = torch.from_numpy(np.ascontiguousarray(b.T)).cuda().t()
    C = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
    ctx.gemm(A, B, EmuConfig(n_moduli=14), C)
    replays = ctx.k3_replays(reset=True)
    want = oracle.gemm(a, b, 14, 0)
    got = C.cpu().numpy()
    assert np.array_equal(got.view(np.int64), want.view(np.int64))
    assert replays < m * n // 1000


@pytest.mark.parametrize("shape", [(128, 4, 96), (256, 12, 300), (640, 36, 1000), (1024, 64, 257), (384, 8, 150),
                                   (512, 40, 600)])
@pytest.mark.parametrize("N", [8, 14, 20])
@pytest.mark.parametrize("ab", [False, True])
def test_k3_full_tiles(oracle, shape, N, ab):
    """Shapes of whole 128-row x 4-column K3 tiles (m % 128 == 0, n % 4 == 0):
    the full-tile instantiation of the column-tiled K3 (no bounds checks, int4
    loads of the column exponents); with n % 8 == 0 also the 8-column tiles
    (OZK_K3_TILE=8 in the variant sweep). N = 8: exact C2; 14: the interval;
    20: 24-plane boxes. Bit-exact against the oracle, with and without alpha/beta
    (the variant sweep reruns this under replay-all and with OZK_K3_FULL=0)."""
    torch = pytest.importorskip("torch")
    from paper_2508_03984_b200 import Context, EmuConfig, gen_matrix

    m, n, k = shape
    a = gen_matrix(m, k, 1.0, 21 + N)
    b = gen_matrix(k, n, 1.0, 22 + N)
    c0 = gen_matrix(m, n, 0.5, 23)
    alpha, beta = (-1.25, 0.5) if ab else (1.0, 0.0)
    want = oracle.gemm(a, b, N, 0)
    if ab:
        want = alpha * want + beta * c0
    A = torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()
    B = torch.from_numpy(np.ascontiguousarray(b.T)).cuda().t()
    C = torch.from_numpy(np.ascontiguousarray(c0.T)).cuda().t()
    Context(0).gemm(A, B, EmuConfig(n_moduli=N), C, alpha=alpha, beta=beta)
    got = C.cpu().numpy()
    assert np.array_equal(got.view(np.int64), want.view(np.int64))
