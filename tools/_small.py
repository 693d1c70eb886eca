import torch, sys
sys.path.insert(0, '.')
from paper_2508_03984_b200 import Context, EmuConfig, ScaleMode
n = int(sys.argv[1])
ctx = Context(0); ctx.set_stream(torch.cuda.current_stream().cuda_stream)
A = (torch.rand((n, n), device="cuda", dtype=torch.float64) - 0.5).t()
B = (torch.rand((n, n), device="cuda", dtype=torch.float64) - 0.5).t()
C = torch.empty((n, n), device="cuda", dtype=torch.float64).t()
for mode in (ScaleMode.Fast, ScaleMode.Accurate):
    for _ in range(2):
        ctx.gemm(A, B, EmuConfig(n_moduli=14, mode=mode), C)
torch.cuda.synchronize()
