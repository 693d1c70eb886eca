"""Host<->device copy rates the e2e path is bounded by (pinned memory):
contiguous H2D / D2H, pitched 2D copies with 2/4/16/64 KB runs, and H2D+D2H
concurrently (full duplex)."""
import json

import torch
from cuda.bindings import runtime as rt


def main():
    n = 16384
    host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    host2 = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    dev = torch.empty((n, n), dtype=torch.float64, device="cuda")
    dev2 = torch.empty((n, n), dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}

    def timed(fn, nbytes, reps=3):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return nbytes * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9

    nb = n * n * 8
    out["h2d_GBs"] = timed(lambda: dev.copy_(host, non_blocking=True), nb)
    out["d2h_GBs"] = timed(lambda: host.copy_(dev, non_blocking=True), nb)

    def duplex():
        ev = torch.cuda.Event()
        ev.record()
        s1.wait_event(ev)
        s2.wait_event(ev)
        with torch.cuda.stream(s1):
            dev.copy_(host, non_blocking=True)
        with torch.cuda.stream(s2):
            host2.copy_(dev2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)

    out["duplex_each_GBs"] = timed(duplex, nb)
    for run_kb in (2, 4, 16, 64):
        rows = run_kb * 1024 // 8  # rows of a column-major row block
        blocks = n // rows
        # copy row block by row block: each a pitched 2D copy (run = rows*8 bytes, n runs)
        pitch = n * 8
        s = torch.cuda.current_stream().cuda_stream

        def pitched():
            for b in range(blocks):
                off = b * rows * 8
                rt.cudaMemcpy2DAsync(dev.data_ptr() + off, pitch, host.data_ptr() + off, pitch, rows * 8, n,
                                     rt.cudaMemcpyKind.cudaMemcpyHostToDevice, s)

        out[f"h2d_pitched_{run_kb}KB_GBs"] = timed(pitched, nb, reps=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
