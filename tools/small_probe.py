"""Per-call timing at a small size (host wall clock and device events per
call), to find outliers: python tools/small_probe.py [n]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_03984_b200 import Context, EmuConfig, ScaleMode  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    ctx = Context(0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    A = (torch.rand((n, n), device="cuda", dtype=torch.float64) - 0.5).t()
    B = (torch.rand((n, n), device="cuda", dtype=torch.float64) - 0.5).t()
    C = torch.empty((n, n), device="cuda", dtype=torch.float64).t()
    for mode, so in ((ScaleMode.Fast, False), (ScaleMode.Accurate, False), (ScaleMode.Fast, True),
                     (ScaleMode.Accurate, True)):
        cfg = EmuConfig(n_moduli=14, mode=mode, stream_ordered=so)
        for _ in range(3):
            ctx.gemm(A, B, cfg, C)
        torch.cuda.synchronize()
        host, dev = [], []
        for _ in range(40):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(stream)
            ctx.gemm(A, B, cfg, C)
            e1.record(stream)
            torch.cuda.synchronize()
            host.append((time.perf_counter() - t0) * 1e3)
            dev.append(e0.elapsed_time(e1))
        host.sort()
        dev.sort()
        print(f"n={n} {mode.name} async={so}: host ms median {host[20]:.3f} max {host[-1]:.3f}; "
              f"device ms median {dev[20]:.3f} max {dev[-1]:.3f}", flush=True)


if __name__ == "__main__":
    main()
