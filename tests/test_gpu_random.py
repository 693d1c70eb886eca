"""Randomised parity sweep: 64 seeded draws of shape, modulus count, mode,
precision, input dynamic range (incl. zero rows/columns and huge spreads),
transposes and alpha/beta, each through the device API and compared bit for
bit with the oracle (tests/_oracle.py, pinned against the reference's own
sources). The draws are fixed by the seed so a failure reproduces by id."""
import numpy as np
import pytest

from paper_2508_03984_b200 import Context, EmuConfig, Precision, ScaleMode, gen_matrix

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _bits(x):
    x = np.ascontiguousarray(x)
    return x.view(np.int64) if x.dtype == np.float64 else x.view(np.int32)


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t()


def _draw(i):
    r = np.random.default_rng(1000 + i)
    small = r.random() < 0.6
    m, n, k = (int(v) for v in r.integers(1, 300 if small else 1500, size=3))
    if r.random() < 0.3:  # whole 64-row tiles: the vectorised row-statistics path
        m = max(64, m // 64 * 64)
    prec = 1 if r.random() < 0.3 else 0
    N = int(r.integers(2, 21)) if prec == 0 else int(r.integers(2, 13))
    return dict(m=m, n=n, k=k, N=N, prec=prec, mode=int(r.integers(0, 2)), phi=float(r.choice([0.0, 0.5, 1.0, 2.0, 4.0])),
                ta=bool(r.random() < 0.25), tb=bool(r.random() < 0.25), zero_row=bool(r.random() < 0.3),
                ab=bool(r.random() < 0.25), seed=int(r.integers(0, 1 << 30)))


@pytest.mark.parametrize("i", range(64))
def test_random_draw(oracle, i):
    d = _draw(i)
    m, n, k, N, prec = d["m"], d["n"], d["k"], d["N"], d["prec"]
    dt = np.float64 if prec == 0 else np.float32
    a = gen_matrix(m, k, d["phi"], d["seed"], dt)
    b = gen_matrix(k, n, d["phi"], d["seed"] + 1, dt)
    if d["zero_row"]:
        a[m // 2, :] = 0
        b[:, n // 2] = 0
    alpha, beta = (-1.25, 0.5) if d["ab"] else (1.0, 0.0)
    c0 = gen_matrix(m, n, 0.5, d["seed"] + 2, dt)
    want = oracle.gemm(a, b, N, d["mode"], prec=prec)  # FP64 result of the reference
    if d["ab"]:  # the alpha/beta extension: fl(fl(alpha*AB) + fl(beta*C)) in FP64
        want = alpha * want + beta * c0.astype(np.float64)
    if prec == 1:
        want = want.astype(np.float32)
    cfg = EmuConfig(n_moduli=N, mode=ScaleMode(d["mode"]), precision=Precision(prec))
    A = _dev(np.asfortranarray(a.T)) if d["ta"] else _dev(a)  # stored transposed: op(A) = A^T
    B = _dev(np.asfortranarray(b.T)) if d["tb"] else _dev(b)
    C = _dev(c0)
    ctx = Context(0)
    ctx.gemm(A, B, cfg, C, alpha=alpha, beta=beta, trans_a=d["ta"], trans_b=d["tb"])
    torch.cuda.synchronize()
    np.testing.assert_array_equal(_bits(C.cpu().numpy()), _bits(want), err_msg=str(d))
