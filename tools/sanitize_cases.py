"""Small invocations of every kernel family for compute-sanitizer
(tools/sanitize.sh): fast/accurate FP64, FP32 tables, the streamed host
pipeline, k > 2^17 chunks, the int64 bound product (k > 2^19), transposes,
alpha/beta and the stage exports. Each result is checked against the oracle
so a tool that perturbs timing cannot hide a wrong answer."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from _oracle import Oracle  # noqa: E402

from paper_2508_03984_b200 import Context, EmuConfig, Precision, ScaleMode, gen_matrix  # noqa: E402

quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
orc = Oracle()
ctx = Context(0)
bad = 0


def check(tag, got, want):
    global bad
    same = np.array_equal(np.ascontiguousarray(got).view(np.int64), np.ascontiguousarray(want).view(np.int64))
    print(f"{tag}: {'ok' if same else 'MISMATCH'}", flush=True)
    bad += not same


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t()


for (m, n, k) in [(200, 300, 1000), (257, 129, 4100)]:
    a, b = gen_matrix(m, k, 0.5, 1), gen_matrix(k, n, 0.5, 2)
    for mode in (ScaleMode.Fast, ScaleMode.Accurate):
        cfg = EmuConfig(n_moduli=14, mode=mode)
        C = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
        ctx.gemm(dev(a), dev(b), cfg, C)
        check(f"device {m}x{n}x{k} N14 {mode.name}", C.cpu().numpy(), orc.gemm(a, b, 14, int(mode)))
        check(f"host {m}x{n}x{k} N14 {mode.name}", ctx.gemm_host(a, b, cfg), orc.gemm(a, b, 14, int(mode)))
    cfg = EmuConfig(n_moduli=8, mode=ScaleMode.Fast, precision=Precision.Fp32)
    a32, b32 = a.astype(np.float32), b.astype(np.float32)
    check(f"fp32 {m}x{n}x{k} N8", ctx.gemm_host(a32, b32, cfg), orc.gemm(a32, b32, 8, 0, prec=1))
    # transposes + alpha/beta through the column pipeline
    C0 = gen_matrix(m, n, 0.0, 5)
    got = ctx.gemm_host(np.asfortranarray(a.T), b, EmuConfig(n_moduli=14), alpha=0.5, beta=2.0,
                        c=np.asfortranarray(C0.copy()), trans_a=True)
    want = 0.5 * orc.gemm(a, b, 14, 0) + 2.0 * C0
    print(f"transA alpha/beta {m}x{n}x{k}: max dev {np.max(np.abs(got - want)):.3g}", flush=True)

# whole 128-row x 4-column (x 8-column with OZK_K3_TILE=8) K3 tiles: the full-tile instantiation
m, n, k = 256, 64, 300
a, b = gen_matrix(m, k, 1.0, 8), gen_matrix(k, n, 1.0, 9)
for N in (14, 20):
    C = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
    ctx.gemm(dev(a), dev(b), EmuConfig(n_moduli=N), C)
    check(f"full tiles {m}x{n}x{k} N{N}", C.cpu().numpy(), orc.gemm(a, b, N, 0))

if not quick:
    # streamed host pipeline (fast mode, m, n >= 2048)
    m = n = 2048
    k = 512
    a, b = gen_matrix(m, k, 0.5, 3), gen_matrix(k, n, 0.5, 4)
    check("host streamed 2048x2048x512", ctx.gemm_host(a, b, EmuConfig(n_moduli=14)), orc.gemm(a, b, 14, 0))
    # k > 2^17: chunked products (fast) and the int64 bound product (accurate, k > 2^19)
    for (m, n, k, mode) in [(40, 24, (1 << 17) + 33, ScaleMode.Fast), (24, 16, (1 << 19) + 17, ScaleMode.Accurate)]:
        a, b = gen_matrix(m, k, 0.5, 6), gen_matrix(k, n, 0.5, 7)
        check(f"long k {m}x{n}x{k} {mode.name}", ctx.gemm_host(a, b, EmuConfig(n_moduli=14, mode=mode)),
              orc.gemm(a, b, 14, int(mode)))
print("sanitize cases:", "all ok" if not bad else f"{bad} mismatches")
sys.exit(1 if bad else 0)
