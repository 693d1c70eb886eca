"""Device-resident emulated DGEMM throughput across sizes (fast / accurate,
N = 14): where launch and host-sync overheads start to matter."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_03984_b200 import Context, EmuConfig, ScaleMode  # noqa: E402


def main():
    ctx = Context(0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    out = {}
    for n in [int(x) for x in os.environ.get("SIZES", "256,512,1024,2048,4096,8192").split(",")]:
        A = (torch.rand((n, n), device="cuda", dtype=torch.float64) - 0.5).t()
        B = (torch.rand((n, n), device="cuda", dtype=torch.float64) - 0.5).t()
        C = torch.empty((n, n), device="cuda", dtype=torch.float64).t()
        for mode, so in ((ScaleMode.Fast, False), (ScaleMode.Accurate, False), (ScaleMode.Fast, True),
                         (ScaleMode.Accurate, True)):
            cfg = EmuConfig(n_moduli=14, mode=mode, stream_ordered=so)
            for _ in range(3):
                ctx.gemm(A, B, cfg, C)
            torch.cuda.synchronize()
            reps = max(3, min(200, int(2e11 / n ** 3)))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                ctx.gemm(A, B, cfg, C)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            out[f"{n}_{mode.name}{'_async' if so else ''}"] = {"ms": round(ms, 4),
                                                               "tflops": round(2 * n ** 3 / ms / 1e9, 2)}
            if so:  # the same call replayed as a CUDA graph
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
                    ctx.gemm(A, B, cfg, C)
                ctx.set_stream(stream.cuda_stream)
                g.replay()
                torch.cuda.synchronize()
                e0.record(stream)
                for _ in range(reps):
                    g.replay()
                e1.record(stream)
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / reps
                out[f"{n}_{mode.name}_graph"] = {"ms": round(ms, 4), "tflops": round(2 * n ** 3 / ms / 1e9, 2)}
        # native FP64 for reference
        torch.matmul(A, B, out=C)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(reps):
            torch.matmul(A, B, out=C)
        e1.record(stream)
        torch.cuda.synchronize()
        out[f"{n}_fp64"] = round(2 * n ** 3 / (e0.elapsed_time(e1) / reps) / 1e9, 2)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
