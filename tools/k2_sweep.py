"""K2 variant sweep: time the N residue GEMMs alone (ozk_stage_products, uint8
epilogue) at the bench size under different OZK_K2_* knobs. Run under
`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum` to see DRAM
traffic per variant (launch order = the VARIANTS list, `reps` launches each)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_03984_b200 import Context, EmuConfig  # noqa: E402
from paper_2508_03984_b200 import _lib  # noqa: E402

VARIANTS = [
    {"OZK_K2_SYNC": "1", "OZK_K2_GROUP": "8"},
    {"OZK_K2_SYNC": "1", "OZK_K2_GROUP": "4"},
    {"OZK_K2_SYNC": "1", "OZK_K2_GROUP": "12"},
    {"OZK_K2_SYNC": "0"},
]


def main():
    n = int(os.environ.get("SWEEP_N", "16384"))
    n_mod = int(os.environ.get("SWEEP_MODULI", "14"))
    reps = int(os.environ.get("SWEEP_REPS", "3"))
    ctx = Context(0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    m = k = n
    data = os.environ.get("SWEEP_DATA", "random")  # random | zero | small (|x| <= 3): power vs operand toggling
    if data == "zero":
        pa = torch.zeros((n_mod, k, ctx.plane_ld(m)), dtype=torch.int8, device="cuda")
        pb = torch.zeros((n_mod, n, ctx.plane_ld(k)), dtype=torch.int8, device="cuda")
    else:
        lo, hi = (-128, 128) if data == "random" else (-3, 4)
        pa = torch.randint(lo, hi, (n_mod, k, ctx.plane_ld(m)), dtype=torch.int8, device="cuda")
        pb = torch.randint(lo, hi, (n_mod, n, ctx.plane_ld(k)), dtype=torch.int8, device="cuda")
    u = torch.empty((n_mod, n, (m + 15) // 16 * 16), dtype=torch.uint8, device="cuda")
    cfg = EmuConfig(n_moduli=n_mod)
    out = []
    variants = json.loads(os.environ["SWEEP_VARIANTS"]) if "SWEEP_VARIANTS" in os.environ else VARIANTS
    for v in variants:
        os.environ.update(v)
        ctx.stage_products(cfg, m, n, k, pa, pb, _lib.OZK_PRODUCTS_U8, u, u.shape[2])  # warm
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            ctx.stage_products(cfg, m, n, k, pa, pb, _lib.OZK_PRODUCTS_U8, u, u.shape[2])
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out.append({**v, "ms": round(ms, 3), "tops": round(n_mod * 2.0 * m * n * k / ms / 1e9, 1)})
        print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
