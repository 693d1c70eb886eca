"""CPU stand-in for the GPU shard engine (TEST INFRASTRUCTURE): implements
shard_begin / shard_rowmax / shard_end with the oracle, so the multi-process
exchange logic of paper_2508_03984_b200.distributed runs under gloo on CPU
(and shard_stream_begin / _rows / _end, the row-streamed fast-mode path).
Per rank it computes exactly what ozk_shard_begin/_end compute on the GPU:
fast mode scales from A and the local columns; accurate mode the partial row
maxima of Abar*Bbar_local (scaling.cpp:118-148), then the budget from the
all-reduced maxima (scaling.cpp:151-165)."""
import numpy as np
import torch


def _ilogb(x):
    return np.frexp(x)[1] - 1


class CpuShardEngine:
    def __init__(self, oracle, n_moduli):
        self.o = oracle
        self.N = n_moduli

    def shard_begin(self, A, B, cfg):
        self.a = np.asfortranarray(A.numpy())
        self.b = np.asfortranarray(B.numpy())
        self.mode = int(cfg.mode)
        if self.mode == 0:
            self.mu, self.nu = self.o.scale(self.a, self.b, self.N, 0)
            self._rowmax = torch.zeros(self.a.shape[0], dtype=torch.int32)
            return
        amax = np.abs(self.a).max(axis=1)
        bmax = np.abs(self.b).max(axis=0)
        self.ma = np.where(amax != 0, 5 - _ilogb(np.where(amax != 0, amax, 1.0)), 0)
        nb = np.where(bmax != 0, 5 - _ilogb(np.where(bmax != 0, bmax, 1.0)), 0)
        abar = np.ceil(np.ldexp(np.abs(self.a), self.ma[:, None])).astype(np.int64)
        bbar = np.ceil(np.ldexp(np.abs(self.b), nb[None, :])).astype(np.int64)
        cbar = abar @ bbar
        self.amax = amax
        self._rowmax = torch.from_numpy(cbar.max(axis=1).astype(np.int32))
        colmax = cbar.max(axis=0)
        self.nu = np.array([self.o.accurate_exponent(int(c), int(e), self.N) if bm != 0 else 0
                            for c, e, bm in zip(colmax, nb, bmax)], np.int32)

    def shard_rowmax(self):
        return self._rowmax

    def shard_end(self, C, alpha=1.0, beta=0.0):
        assert alpha == 1.0 and beta == 0.0
        if self.mode == 1:
            rm = self._rowmax.numpy()
            self.mu = np.array([self.o.accurate_exponent(int(c), int(e), self.N) if am != 0 else 0
                                for c, e, am in zip(rm, self.ma, self.amax)], np.int32)
        out = self.o.gemm_scaled(self.a, self.b, self.N, self.mu, self.nu)
        C.copy_(torch.from_numpy(np.ascontiguousarray(out.T)).t())

    # ---- row-streamed fast mode: C rows per block of A (mu is row-local) ----
    def shard_stream_begin(self, m, k, B, cfg, C, alpha=1.0, beta=0.0):
        assert int(cfg.mode) == 0 and alpha == 1.0 and beta == 0.0
        self.b = np.asfortranarray(B.numpy())
        self.C = C
        self.rows = 0

    def shard_stream_rows(self, r0, A_rows):
        a = np.asfortranarray(A_rows.numpy())
        out = self.o.gemm(a, self.b, self.N, 0)
        self.C[r0:r0 + a.shape[0]].copy_(torch.from_numpy(np.ascontiguousarray(out.T)).t())
        self.rows += a.shape[0]

    def shard_stream_end(self):
        assert self.rows == self.C.shape[0]
