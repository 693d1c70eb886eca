"""How fast do memory-bound kernels run right after the power-capped K2?
On one stream, stream-ordered (no host sync between the GEMM and the probe):
the SM clock seen by a 50k-cycle spin kernel (torch.cuda._sleep, timed with
events), a 2 GiB device copy, and K3 (ozk_stage_reconstruct) — after the GPU
idled, and immediately after a full 16384^3 N=14 emulated GEMM (K2 leaves the
part at its power cap)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_03984_b200 import Context, EmuConfig  # noqa: E402


def main():
    n, N = 16384, 14
    ctx = Context(0)
    st = torch.cuda.current_stream()
    ctx.set_stream(st.cuda_stream)
    A = torch.randn((n, n), dtype=torch.float64, device="cuda").t()
    B = torch.randn((n, n), dtype=torch.float64, device="cuda").t()
    C = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
    src = torch.empty(1 << 28, dtype=torch.float64, device="cuda")
    dst = torch.empty_like(src)
    U = torch.randint(0, 173, (N, n, n), dtype=torch.uint8, device="cuda")
    mu = torch.zeros(n, dtype=torch.int32, device="cuda")
    cfg = EmuConfig(n_moduli=N, stream_ordered=True)
    spin = 50000

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(st)
        return e

    copy = lambda: dst.copy_(src)
    k3 = lambda: ctx.stage_reconstruct(cfg, n, n, U, n, mu, mu, C)
    for f in (copy, k3):
        f()
    ctx.gemm(A, B, cfg, C)
    torch.cuda.synchronize()
    out = {}
    for name, f in (("copy_2GiB", copy), ("k3", k3)):
        rows = {"idle": [], "after_gemm": []}
        for _ in range(5):
            for when in ("idle", "after_gemm"):
                if when == "idle":
                    torch.cuda.synchronize()
                    time.sleep(1.0)
                else:
                    ctx.gemm(A, B, cfg, C)
                e0 = ev()
                torch.cuda._sleep(spin)
                e1 = ev()
                f()
                e2 = ev()
                torch.cuda._sleep(spin)
                e3 = ev()
                torch.cuda.synchronize()
                rows[when].append((spin / (e0.elapsed_time(e1) * 1e3), e1.elapsed_time(e2),
                                   spin / (e2.elapsed_time(e3) * 1e3)))
        for when, r in rows.items():
            r.sort(key=lambda t: t[1])
            mid = r[len(r) // 2]
            out[f"{name}_{when}"] = {"ms": round(mid[1], 4), "sm_mhz_before": round(mid[0]),
                                     "sm_mhz_after": round(mid[2])}
    for when in ("idle", "after_gemm"):
        out[f"copy_2GiB_{when}"]["TBs"] = round(2 * 2**31 / out[f"copy_2GiB_{when}"]["ms"] / 1e9, 2)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
