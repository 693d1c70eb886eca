"""Parity at BASELINE.json's full sizes (SURVEY §8c "Large-n parity").

The CPU oracle cannot run a 16384^3 emulation in test time, but every entry of
C depends only on row i of A, column j of B and the two scale exponents
(emulator.cpp:34-77). So at the benchmark's own sizes:

* the full mu / nu vectors are checked against the reference's scaling
  (fast: the oracle's `scale` on the whole matrices; accurate: the bound
  product Abar*Bbar computed exactly in FP64 on the GPU -- its entries are
  integers < 2^53, so any summation order is exact -- then the oracle's
  exponent rule, scaling.cpp:151-165, per line), and
* C is checked bit-for-bit on sampled rows x columns (>= 4096 entries,
  including the first/last row and column) against the oracle pipeline run on
  those rows of A and columns of B with the same exponents.

Inputs are the paper's generator (rand-0.5)*exp(phi*randn) drawn on the
device (torch Philox); test data only.
"""
import numpy as np
import pytest

from paper_2508_03984_b200 import EmuConfig, Precision, ScaleMode

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _bits(x):
    return np.ascontiguousarray(x).view(np.int64)


def _gen(rows, cols, phi, seed, dtype):
    g = torch.Generator(device="cuda").manual_seed(seed)
    r = 1.0 - torch.rand((cols, rows), generator=g, device="cuda", dtype=torch.float64)
    x = r - 0.5
    if phi:
        x = x * torch.exp(phi * torch.randn((cols, rows), generator=g, device="cuda", dtype=torch.float64))
    return x.to(dtype).t()  # (rows, cols), column-major


def _host(t):
    return np.asfortranarray(t.cpu().numpy())


def _ilogb(t):
    return torch.frexp(t)[1] - 1


def _accurate_exponents(oracle, A, B, N):
    """mu/nu of scale_accurate (scaling.cpp:101-167), bound GEMM exact in FP64"""
    a, b = A.double().abs(), B.double().abs()
    amax, bmax = a.amax(dim=1), b.amax(dim=0)
    ma = torch.where(amax != 0, 5 - _ilogb(torch.where(amax != 0, amax, 1.0)), 0)
    nb = torch.where(bmax != 0, 5 - _ilogb(torch.where(bmax != 0, bmax, 1.0)), 0)
    abar = torch.ceil(torch.ldexp(a, ma[:, None].double()))
    bbar = torch.ceil(torch.ldexp(b, nb[None, :].double()))
    assert abar.max() <= 64 and bbar.max() <= 64
    cbar = abar @ bbar  # integers <= 64*64*k < 2^53: exact in any order
    rowmax = cbar.amax(dim=1).long().cpu().numpy()
    colmax = cbar.amax(dim=0).long().cpu().numpy()
    prec = 1 if A.dtype == torch.float32 else 0
    cs = oracle.constants(N, prec)
    f = oracle.lib.ozo_accurate_exponent
    import ctypes as C

    def line(cmax, base, nz):
        return np.array([f(int(c), int(e), C.byref(cs)) if z else 0 for c, e, z in zip(cmax, base, nz)], np.int32)

    return (line(rowmax, ma.cpu().numpy(), (amax != 0).cpu().numpy()),
            line(colmax, nb.cpu().numpy(), (bmax != 0).cpu().numpy()))


def _sample(count, size, rng):
    inner = rng.choice(np.arange(1, size - 1), count - 2, replace=False)
    return np.array(sorted(set(inner.tolist()) | {0, size - 1}))


CASES = [
    # (m, n, k, N, mode, phi, precision)  -- BASELINE.json configs[1], [2], [4]
    (16384, 16384, 16384, 14, ScaleMode.Fast, 0.5, Precision.Fp64),
    (16384, 16384, 16384, 14, ScaleMode.Accurate, 0.5, Precision.Fp64),
    (16384, 16384, 16384, 12, ScaleMode.Fast, 0.0, Precision.Fp64),
    (16384, 16384, 16384, 20, ScaleMode.Accurate, 4.0, Precision.Fp64),
    (16384, 16384, 16384, 8, ScaleMode.Fast, 0.5, Precision.Fp32),
    (16384, 16384, 16384, 10, ScaleMode.Accurate, 1.0, Precision.Fp32),
    (8192, 8192, 65536, 14, ScaleMode.Fast, 0.5, Precision.Fp64),
    (32768, 32768, 32768, 14, ScaleMode.Fast, 0.5, Precision.Fp64),  # configs[3] per-GPU problem at 1 GPU
    # every other point bench.py times (round 2)
    (16384, 16384, 16384, 15, ScaleMode.Fast, 0.5, Precision.Fp64),
    (16384, 16384, 16384, 15, ScaleMode.Accurate, 0.5, Precision.Fp64),
    (16384, 16384, 16384, 16, ScaleMode.Fast, 0.5, Precision.Fp64),
    (16384, 16384, 16384, 16, ScaleMode.Accurate, 0.5, Precision.Fp64),
    (16384, 16384, 16384, 18, ScaleMode.Fast, 0.5, Precision.Fp64),
    (16384, 16384, 16384, 18, ScaleMode.Accurate, 0.5, Precision.Fp64),
    (16384, 16384, 16384, 6, ScaleMode.Fast, 0.5, Precision.Fp32),
    (16384, 16384, 16384, 7, ScaleMode.Accurate, 0.5, Precision.Fp32),
    (16384, 16384, 16384, 9, ScaleMode.Fast, 0.5, Precision.Fp32),
    (16384, 16384, 16384, 9, ScaleMode.Accurate, 0.5, Precision.Fp32),
    (8192, 8192, 65536, 14, ScaleMode.Accurate, 0.5, Precision.Fp64),
]


@pytest.mark.parametrize("m,n,k,N,mode,phi,prec", CASES)
def test_full_size_sampled_parity(ctx, oracle, m, n, k, N, mode, phi, prec):
    dt = torch.float32 if prec == Precision.Fp32 else torch.float64
    A = _gen(m, k, phi, 1, dt)
    B = _gen(k, n, phi, 2, dt)
    cfg = EmuConfig(n_moduli=N, mode=mode, precision=prec)
    Cg = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
    ctx.gemm(A, B, cfg, Cg)
    mu = torch.zeros(m, dtype=torch.int32, device="cuda")
    nu = torch.zeros(n, dtype=torch.int32, device="cuda")
    ctx.stage_scale(A, B, cfg, mu, nu)
    mu, nu = mu.cpu().numpy(), nu.cpu().numpy()

    if mode == ScaleMode.Fast:
        wmu, wnu = oracle.scale(_host(A), _host(B), N, 0, int(prec))
    else:
        wmu, wnu = _accurate_exponents(oracle, A, B, N)
    np.testing.assert_array_equal(mu, wmu)
    np.testing.assert_array_equal(nu, wnu)

    rng = np.random.default_rng(m + k + N)
    rows, cols = _sample(64, m, rng), _sample(64, n, rng)
    a_rows = _host(A[torch.from_numpy(rows).cuda(), :])
    b_cols = _host(B[:, torch.from_numpy(cols).cuda()])
    want = oracle.gemm_scaled(a_rows, b_cols, N, wmu[rows], wnu[cols], prec=int(prec))
    got = Cg[torch.from_numpy(rows).cuda()][:, torch.from_numpy(cols).cuda()].cpu().numpy()
    assert got.size >= 4096
    np.testing.assert_array_equal(_bits(got), _bits(want))


def _gen_chunked(rows, cols, phi, seed, chunk=2048):
    """the paper's generator drawn column block by column block into one
    preallocated column-major FP64 matrix (no full-size temporaries)"""
    out = torch.empty((cols, rows), dtype=torch.float64, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(seed)
    for j0 in range(0, cols, chunk):
        j1 = min(cols, j0 + chunk)
        blk = out[j0:j1]
        torch.rand(blk.shape, generator=g, device="cuda", dtype=torch.float64, out=blk)
        blk.neg_().add_(0.5)  # (1 - r) - 0.5 with r in [0, 1)
        if phi:
            blk.mul_(torch.exp(phi * torch.randn(blk.shape, generator=g, device="cuda", dtype=torch.float64)))
    return out.t()


def test_65536_single_gpu_sampled_parity(ctx, oracle):
    """BASELINE configs[3] at one GPU: DGEMM 65536^3, N = 14, fast mode. A, B and
    C alone take 103 GB, the full workspace would take 180 GB more, so the call
    runs in panels under the automatic workspace limit. Fast-mode mu_i depends
    on row i of A only and nu_j on column j of B only (scaling.cpp:58-99), so
    the reference exponents of sampled rows/columns come from those rows and
    columns alone; C is compared bit for bit on 64 x 64 sampled entries."""
    import gc

    n = 65536
    N = 14
    gc.collect()  # contexts of earlier tests release their workspace
    ctx.release_workspace()
    torch.cuda.empty_cache()
    A = _gen_chunked(n, n, 0.5, 1)
    B = _gen_chunked(n, n, 0.5, 2)
    C = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
    torch.cuda.empty_cache()
    cfg = EmuConfig(n_moduli=N, mode=ScaleMode.Fast)
    # the footprint target: caller's A, B, C + workspace <= 160 GB
    ctx.set_workspace_limit(int(158e9) - torch.cuda.memory_allocated())
    free, total = torch.cuda.mem_get_info()
    print(f"before the call: {free / 1e9:.1f} of {total / 1e9:.1f} GB free")
    ctx.gemm(A, B, cfg, C)
    torch.cuda.synchronize()
    plan = ctx.last_plan
    # this call's footprint: the caller's A, B, C plus the handle's workspace
    # (other handles of the test session may hold memory of their own)
    used_gb = (torch.cuda.memory_allocated() + ctx.workspace_bytes) / 1e9
    print(f"65536^3 N=14 fast: plan {plan}, A+B+C+workspace {used_gb:.1f} GB "
          f"(workspace {ctx.workspace_bytes / 1e9:.1f} GB)")
    assert plan["panels"] > 1
    assert used_gb <= 160.0
    mu = torch.zeros(n, dtype=torch.int32, device="cuda")
    nu = torch.zeros(n, dtype=torch.int32, device="cuda")
    ctx.stage_scale(A, B, cfg, mu, nu)
    rng = np.random.default_rng(65536)
    rows, cols = _sample(64, n, rng), _sample(64, n, rng)
    ri, ci = torch.from_numpy(rows).cuda(), torch.from_numpy(cols).cuda()
    a_rows = _host(A[ri, :])
    b_cols = _host(B[:, ci])
    wmu, wnu = oracle.scale(a_rows, b_cols, N, 0, 0)  # row/column-local in fast mode
    np.testing.assert_array_equal(mu[ri].cpu().numpy(), wmu)
    np.testing.assert_array_equal(nu[ci].cpu().numpy(), wnu)
    want = oracle.gemm_scaled(a_rows, b_cols, N, wmu, wnu)
    got = C[ri][:, ci].cpu().numpy()
    np.testing.assert_array_equal(_bits(got), _bits(want))
    ctx.set_workspace_limit(0)
    ctx.release_workspace()
    del A, B, C
    torch.cuda.empty_cache()
