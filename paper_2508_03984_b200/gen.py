"""Synthetic inputs: the paper's generator ``(rand - 0.5) * exp(phi * randn)``.

SPEC.md:400-408 (gen_matrix) / PAPER.md §5: rand uniform on (0, 1], randn
standard normal, seeded and deterministic. Frozen choice (SPEC.md:422 leaves
it open): numpy's Philox bit generator keyed by ``seed``; ``rand = 1 - U[0,1)``
and ``randn`` from ``Generator.standard_normal``; both drawn as full
column-major (Fortran-order) blocks, rand first. phi = 0 gives U(-0.5, 0.5].
"""
from __future__ import annotations

import numpy as np


def gen_matrix(rows: int, cols: int, phi: float = 0.5, seed: int = 1, dtype=np.float64) -> np.ndarray:
    rng = np.random.Generator(np.random.Philox(seed))
    rand = 1.0 - rng.random((cols, rows))          # (0, 1]
    if phi == 0.0:
        x = rand - 0.5
    else:
        x = (rand - 0.5) * np.exp(phi * rng.standard_normal((cols, rows)))
    return np.asarray(x.T, dtype=dtype, order="F")


def gen_int_matrix(rows: int, cols: int, bound: int, seed: int = 1, dtype=np.float64) -> np.ndarray:
    """Integer-valued matrix with entries uniform in [-bound, bound] (exactness tests)."""
    rng = np.random.Generator(np.random.Philox(seed))
    x = rng.integers(-bound, bound + 1, size=(cols, rows))
    return np.asarray(x.T, dtype=dtype, order="F")
