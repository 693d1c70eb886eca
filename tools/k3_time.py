"""Time K3 (ozk_stage_reconstruct) alone at the bench size: N uint8 planes of
m x n -> FP64 C. Knob: OZK_K3_ROWS (4 or 8 rows per thread)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_03984_b200 import Context, EmuConfig, Precision  # noqa: E402


def main():
    n = int(os.environ.get("K3_N", "16384"))
    reps = int(os.environ.get("K3_REPS", "10"))
    out = {"rows": os.environ.get("OZK_K3_ROWS", "default")}
    ctx = Context(0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    for N in [int(x) for x in os.environ.get("K3_MODS", "8,14,20").split(",")]:
        ldu = (n + 15) // 16 * 16
        U = torch.randint(0, 173, (N, n, ldu), dtype=torch.uint8, device="cuda")
        mu = torch.zeros(n, dtype=torch.int32, device="cuda")
        prec = int(os.environ.get("K3_PREC", "0"))  # 1: FP32 tables (SGEMM), FP32 C
        C = torch.empty((n, n), dtype=torch.float32 if prec else torch.float64, device="cuda").t()
        cfg = EmuConfig(n_moduli=N, precision=Precision(prec))
        ctx.stage_reconstruct(cfg, n, n, U, ldu, mu, mu, C)
        torch.cuda.synchronize()
        ctx.k3_replays(reset=True)  # start counting
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            ctx.stage_reconstruct(cfg, n, n, U, ldu, mu, mu, C)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out[f"N{N}_ms"] = round(ms, 3)
        out[f"N{N}_replays_per_call"] = ctx.k3_replays(reset=True) / reps
        out[f"N{N}_TBs"] = round((N + (4 if prec else 8)) * n * n / ms / 1e9, 2)
        del U
    print(json.dumps(out))


if __name__ == "__main__":
    main()
