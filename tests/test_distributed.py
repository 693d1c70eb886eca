"""Multi-process column sharding (world_size 2, gloo, CPU): the exchange logic
of paper_2508_03984_b200.distributed — A broadcast from rank 0, the accurate
row-bound all-reduce(MAX) — reproduces the single-process result bit for bit.
The per-rank compute is the oracle stand-in (tests/_shard_cpu.py); the GPU
engine behind the same three calls is ozk_shard_begin/_rowmax/_end."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, n, k, N, mode, phi, outdir, row_block):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _oracle import Oracle
    from _shard_cpu import CpuShardEngine

    from paper_2508_03984_b200 import EmuConfig, ScaleMode
    from paper_2508_03984_b200.distributed import column_shard, gemm_sharded
    from paper_2508_03984_b200.gen import gen_matrix

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    a = gen_matrix(m, k, phi, 1)
    b = gen_matrix(k, n, phi, 2)
    if rank != 0:
        a = np.zeros_like(a, order="F")  # only the root's A is real: the broadcast must deliver it
    A = torch.from_numpy(np.ascontiguousarray(a.T)).t()
    j0, nj = column_shard(n, world, rank)
    B = torch.from_numpy(np.ascontiguousarray(b[:, j0:j0 + nj].T)).t()
    C = torch.zeros((nj, m), dtype=torch.float64).t()
    gemm_sharded(CpuShardEngine(Oracle(), N), A, B, EmuConfig(n_moduli=N, mode=ScaleMode(mode)), C,
                 row_block=row_block)
    np.save(os.path.join(outdir, f"c{rank}.npy"), C.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("mode,row_block", [(0, None), (0, 8), (1, None), (1, 8)])
@pytest.mark.parametrize("m,n,k,N,phi", [(33, 37, 50, 14, 0.5), (20, 9, 70, 17, 2.0), (100, 12, 40, 14, 1.0)])
def test_sharded_matches_single_process(tmp_path, oracle, mode, row_block, m, n, k, N, phi):
    """row_block=8, fast mode: A streamed in row blocks of 16 rows, one
    async broadcast per block (accurate mode ignores it: mu needs all columns);
    m = 100 gives 7 blocks, so the ring of 3 pack buffers wraps"""
    from paper_2508_03984_b200.gen import gen_matrix

    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), m, n, k, N, mode, phi, str(tmp_path), row_block), nprocs=world,
                       start_method="spawn")
    got = np.concatenate([np.load(tmp_path / f"c{r}.npy") for r in range(world)], axis=1)
    want = oracle.gemm(gen_matrix(m, k, phi, 1), gen_matrix(k, n, phi, 2), N, mode)
    np.testing.assert_array_equal(got.view(np.int64), want.view(np.int64))


def test_column_shard_partition():
    from paper_2508_03984_b200.distributed import column_shard

    for n, w in ((37, 2), (16384, 8), (5, 8)):
        blocks = [column_shard(n, w, r) for r in range(w)]
        assert sum(nj for _, nj in blocks) == n
        assert all(blocks[r][0] + blocks[r][1] == blocks[r + 1][0] for r in range(w - 1))


def test_row_blocks_cover():
    from paper_2508_03984_b200.distributed import row_blocks

    for m in (1, 7, 512, 2048, 16384, 16385):
        for rb in (1, 8, 2048):
            blocks = row_blocks(m, rb)
            assert blocks[0][0] == 0 and all(mr >= 1 for _, mr in blocks)
            assert all(a[0] + a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
            assert all(r0 % 16 == 0 for r0, _ in blocks)
            assert blocks[-1][0] + blocks[-1][1] == m
