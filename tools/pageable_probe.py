"""What the reference-facing host call can get from PAGEABLE memory (a
crtgemm Matrix<T> is a std::vector): the driver's own staging for pageable
cudaMemcpy, cudaHostRegister cost, and multi-threaded host memcpy into pinned
memory (the staging-ring alternative). Prints one JSON line."""
import json
import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch
from cuda.bindings import runtime as rt

nb = 2 << 30  # 2 GiB
src = np.ones(nb // 8)
dev = torch.empty(nb // 8, dtype=torch.float64, device="cuda")
out = {"host_cores": os.cpu_count()}


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


hsrc = torch.from_numpy(src)
out["pageable_h2d_GBs"] = nb / t(lambda: dev.copy_(hsrc)) / 1e9
dst = np.empty_like(src)
hdst = torch.from_numpy(dst)
out["pageable_d2h_GBs"] = nb / t(lambda: hdst.copy_(dev)) / 1e9


def reg():
    e, = rt.cudaHostRegister(src.ctypes.data, nb, 0)
    assert e == rt.cudaError_t.cudaSuccess, e
    e, = rt.cudaHostUnregister(src.ctypes.data)


out["host_register_GBs"] = nb / t(reg, 2) / 1e9
rt.cudaHostRegister(src.ctypes.data, nb, 0)
out["registered_h2d_GBs"] = nb / t(lambda: dev.copy_(hsrc, non_blocking=True)) / 1e9
rt.cudaHostUnregister(src.ctypes.data)
pin = torch.empty(nb // 8, dtype=torch.float64, pin_memory=True).numpy()
for th in (1, 4, 8, 16, 32):
    if th > 2 * (os.cpu_count() or 1):
        break
    parts = np.array_split(np.arange(src.size), th)
    bounds = [(p[0], p[-1] + 1) for p in parts]
    with ThreadPoolExecutor(th) as ex:
        def cp():
            list(ex.map(lambda b: np.copyto(pin[b[0]:b[1]], src[b[0]:b[1]]), bounds))
        out[f"memcpy_to_pinned_{th}thr_GBs"] = nb / t(cp) / 1e9
print(json.dumps(out))
