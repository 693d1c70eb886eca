"""Does K3 (reconstruction) run for free next to K2 (residue GEMMs)?
Two handles on two streams driven from two host threads (the stage calls
block on their own stream): K2 alone, K3 alone, then K2 with K3 looping
beside it. Synthetic planes at 16384^2, N = 14."""
import json
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_03984_b200 import Context, EmuConfig, _lib  # noqa: E402

n = int(os.environ.get("N_SIZE", "16384"))
N = 14
cfg = EmuConfig(n_moduli=N)
ld = (n + 15) // 16 * 16
dev = "cuda"
pa = torch.randint(-127, 128, (N, n, ld), dtype=torch.int8, device=dev)
pb = torch.randint(-127, 128, (N, n, ld), dtype=torch.int8, device=dev)
U2 = torch.empty((N, n, ld), dtype=torch.uint8, device=dev)
U3 = torch.randint(0, 173, (N, n, ld), dtype=torch.uint8, device=dev)
mu = torch.zeros(n, dtype=torch.int32, device=dev)
C3 = torch.empty((n, n), dtype=torch.float64, device=dev).t()
s2, s3 = torch.cuda.Stream(), torch.cuda.Stream()
c2, c3 = Context(0), Context(0)
c2.set_stream(s2.cuda_stream)
c3.set_stream(s3.cuda_stream)


def k2():
    c2.stage_products(cfg, n, n, n, pa, pb, _lib.OZK_PRODUCTS_U8, U2, ld)


def k3():
    c3.stage_reconstruct(cfg, n, n, U3, ld, mu, mu, C3)


for f in (k2, k3):
    f()
out = {}
t = time.perf_counter()
for _ in range(4):
    k2()
out["k2_alone_ms"] = (time.perf_counter() - t) / 4 * 1e3
t = time.perf_counter()
for _ in range(40):
    k3()
out["k3_alone_ms"] = (time.perf_counter() - t) / 40 * 1e3
stop = threading.Event()
count = [0]


def loop3():
    while not stop.is_set():
        k3()
        count[0] += 1


th = threading.Thread(target=loop3)
th.start()
time.sleep(0.05)
c0 = count[0]
t = time.perf_counter()
for _ in range(4):
    k2()
dt = time.perf_counter() - t
c1 = count[0]
stop.set()
th.join()
out["k2_with_k3_ms"] = dt / 4 * 1e3
out["k3_done_during"] = c1 - c0
out["k3_equiv_ms_during_k2"] = (c1 - c0) * out["k3_alone_ms"] / 4
print(json.dumps(out))
