"""K2 with the moduli-inner schedule (OZK_K2_ORDER=1) — the schedule a K3
fused into K2's epilogue would need, kept as the measured prototype of
SURVEY §8f item 3 — must give the same products: only the order
of the (modulus, tile) work items changes. The knob is read per launch."""
import numpy as np
import pytest

from paper_2508_03984_b200 import EmuConfig, ScaleMode, gen_matrix

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.mark.parametrize("m,n,k,N", [(300, 500, 1000, 14), (1024, 1300, 700, 8), (2000, 2100, 513, 20)])
@pytest.mark.parametrize("mode", [ScaleMode.Fast, ScaleMode.Accurate])
def test_k2_moduli_inner_order(oracle, monkeypatch, m, n, k, N, mode):
    from paper_2508_03984_b200 import gemm_emulated

    monkeypatch.setenv("OZK_K2_ORDER", "1")
    a = gen_matrix(m, k, 0.5, 81)
    b = gen_matrix(k, n, 0.5, 82)
    got = gemm_emulated(a, b, EmuConfig(n_moduli=N, mode=mode)).c
    want = oracle.gemm(a, b, N, int(mode))
    np.testing.assert_array_equal(got.view(np.int64), want.view(np.int64))
