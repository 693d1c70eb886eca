"""The real GPU engine across processes: two ranks on cuda:0 (one B200 in this
run), torch.distributed with gloo carrying CUDA tensors, each rank driving its
own Context through paper_2508_03984_b200.distributed.gemm_sharded — the
row-streamed A broadcast (ring of pack buffers, async broadcasts, the compute
stream waiting per block), the whole-A broadcast, and the accurate-mode
all-reduce(MAX) of the device row maxima. Only rank 0's A is real (rank 1
starts from zeros), and the concatenated column shards must equal the oracle
bit for bit."""
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, n, k, N, mode, phi, outdir, row_block, reps):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from paper_2508_03984_b200 import Context, EmuConfig, ScaleMode
    from paper_2508_03984_b200.distributed import column_shard, gemm_sharded
    from paper_2508_03984_b200.gen import gen_matrix

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    ctx = Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    a = gen_matrix(m, k, phi, 1)
    b = gen_matrix(k, n, phi, 2)
    if rank != 0:
        a = np.zeros_like(a, order="F")  # the broadcast must deliver the root's A
    A = torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()
    j0, nj = column_shard(n, world, rank)
    B = torch.from_numpy(np.ascontiguousarray(b[:, j0:j0 + nj].T)).cuda().t()
    C = torch.zeros((nj, m), dtype=torch.float64, device="cuda").t()
    for _ in range(reps):  # repeated calls reuse the handle's workspace and the ring
        gemm_sharded(ctx, A, B, EmuConfig(n_moduli=N, mode=ScaleMode(mode)), C, row_block=row_block)
    torch.cuda.synchronize()
    np.save(os.path.join(outdir, f"c{rank}.npy"), C.cpu().numpy())
    ctx.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode,row_block", [(0, 256), (0, None), (1, None)])
@pytest.mark.parametrize("m,n,k,N,phi", [(1700, 900, 600, 14, 0.5), (300, 41, 3000, 16, 2.0)])
def test_gpu_sharded_two_processes(tmp_path, oracle, mode, row_block, m, n, k, N, phi):
    import torch.multiprocessing as mp

    from paper_2508_03984_b200.gen import gen_matrix

    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), m, n, k, N, mode, phi, str(tmp_path), row_block, 2),
                       nprocs=world, start_method="spawn")
    got = np.concatenate([np.load(tmp_path / f"c{r}.npy") for r in range(world)], axis=1)
    want = oracle.gemm(gen_matrix(m, k, phi, 1), gen_matrix(k, n, phi, 2), N, mode)
    np.testing.assert_array_equal(got.view(np.int64), want.view(np.int64))
