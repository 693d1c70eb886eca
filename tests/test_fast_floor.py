"""The fast-mode exponent floor near integer budgets (scaling.cpp:45-56).

y = pp_fast - max(1, 0.51 log2 ub) is floored; the reference evaluates log2
with glibc. The GPU evaluates lines whose y lies near an integer in the
reference's sequential order and takes the floor from a host-built step table
(api.cu fast_floor_table) instead of a device log2, so CUDA's and glibc's log2
can never disagree on it. CPU: the table equals the reference expression
(recomputed here in Python doubles over glibc's log2) at random points and on
both sides of every step. GPU: rows and columns whose sequential sum of
squares puts ub on either side of each step give the reference's exponents.
"""
import ctypes
import math

import numpy as np
import pytest

from paper_2508_03984_b200 import Precision, build_constants
from paper_2508_03984_b200 import _lib

_libm = ctypes.CDLL("libm.so.6")
_libm.log2.restype = ctypes.c_double
_libm.log2.argtypes = [ctypes.c_double]


def ref_floor(pp, ub):
    """scaling.cpp:50-52 in IEEE doubles, glibc log2"""
    t = max(1.0, 0.51 * _libm.log2(ub))
    return math.floor(float(np.float32(pp)) - t)


def steps(pp, hi=2.0 ** 40):
    """(threshold, floor below, floor at) for every step of ref_floor over [1, hi]"""
    out = []
    lo = np.float64(1.0).view(np.int64)
    top = np.float64(hi).view(np.int64)
    f = ref_floor(pp, 1.0)
    while ref_floor(pp, float(np.int64(top).view(np.float64))) < f:
        a, b = int(lo), int(top)
        while b - a > 1:
            mid = (a + b) // 2
            if ref_floor(pp, float(np.int64(mid).view(np.float64))) >= f:
                a = mid
            else:
                b = mid
        t = float(np.int64(b).view(np.float64))
        out.append((t, f, ref_floor(pp, t)))
        f = ref_floor(pp, t)
        lo = b
    return out


def _tables():
    for N in range(2, 21):
        yield build_constants(N, Precision.Fp64).pp_fast
    for N in range(2, 19):
        yield build_constants(N, Precision.Fp32).pp_fast


def test_table_equals_reference_expression():
    L = _lib.load()
    rng = np.random.default_rng(5)
    for pp in sorted(set(_tables())):
        for t, below, at in steps(pp):
            prev = float(np.nextafter(t, 0.0))
            assert L.ozk_fast_floor(pp, t, 1) == at == ref_floor(pp, t)
            assert L.ozk_fast_floor(pp, prev, 1) == below == ref_floor(pp, prev)
        for ub in np.exp2(rng.uniform(0, 40, 2000)):
            assert L.ozk_fast_floor(pp, float(ub), 1) == ref_floor(pp, float(ub))


def _sum_of_squares_line(s, k):
    """k powers of two (and zeros) whose squares sum to s exactly in any order,
    the largest element 1.0 (so g = ilogb(max) = 0): s = I + sum_e 2^-e"""
    I = int(math.floor(s))
    frac = s - I
    vals = [1.0] * I
    e = 1
    while frac > 0:
        bit = 2.0 ** -e
        if frac >= bit:
            frac -= bit
            if e % 2 == 0:
                vals.append(2.0 ** (-e // 2))
            else:
                vals += [2.0 ** (-(e + 1) // 2)] * 2
        e += 1
    assert len(vals) <= k and e < 200
    line = np.zeros(k)
    line[:len(vals)] = vals
    np.random.default_rng(len(vals)).shuffle(line)
    return line


def _lowest_bit_even(x):
    """the lowest set bit of x is 2^L with L >= 0 or L even: then x is a sum of
    squares of powers of two whose every partial sum is exact (an odd bit 2^-e
    is two squares 2^-(e+1), which must stay inside the 53-bit window)"""
    m, e = math.frexp(x)
    M, L = int(m * 2 ** 53), e - 53
    while M % 2 == 0:
        M //= 2
        L += 1
    return L >= 0 or L % 2 == 0


def _adversarial_sums(pp, k):
    """sequential sums s whose ub = fl(s (1 + 2 (k+2) 2^-53)) sits just below and
    at each step of the floor reachable with s <= k / 2 (within a few ulps)"""
    factor = 1.0 + 2.0 * (k + 2) * 2.0 ** -53
    out = []
    for t, _, _ in steps(pp):
        if t > k / 2:
            break
        s = t / factor
        below = at = None
        for d in range(-16, 17):
            c = float(np.float64(s) + d * np.spacing(np.float64(s)))
            if not _lowest_bit_even(c):
                continue
            ub = c * factor
            if ub < t:
                below = c
            elif at is None:
                at = c
        out += [x for x in (below, at) if x is not None and x >= 1.0]
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("N,k", [(14, 4096), (12, 65536), (20, 20000)])
def test_gpu_exponents_at_floor_steps(ctx, ref, N, k):
    torch = pytest.importorskip("torch")
    from paper_2508_03984_b200 import EmuConfig, ScaleMode

    pp = build_constants(N).pp_fast
    sums = _adversarial_sums(pp, k)
    assert len(sums) >= 6
    a = np.asfortranarray(np.stack([_sum_of_squares_line(s, k) for s in sums]))  # rows of A
    b = np.asfortranarray(a.T.copy())                                              # columns of B
    mu_ref, nu_ref = ref.scale(a, b, N, 0)
    A = torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()
    B = torch.from_numpy(np.ascontiguousarray(b.T)).cuda().t()
    mu = torch.zeros(a.shape[0], dtype=torch.int32, device="cuda")
    nu = torch.zeros(b.shape[1], dtype=torch.int32, device="cuda")
    ctx.stage_scale(A, B, EmuConfig(n_moduli=N, mode=ScaleMode.Fast), mu, nu)
    np.testing.assert_array_equal(mu.cpu().numpy(), np.log2(mu_ref).astype(np.int32))
    np.testing.assert_array_equal(nu.cpu().numpy(), np.log2(nu_ref).astype(np.int32))
    # the pairs straddle the steps: both floors occur
    assert len(set(np.log2(mu_ref).astype(int).tolist())) >= 3
