"""Multi-process (gloo, world_size 2, CPU) coverage of the sharded assembly logic:
balanced row ranges tile the upper triangle exactly, and row blocks computed
independently per rank (CPU oracle standing in for each rank's GPU) reassemble
into the single-process matrix; the max-over-ranks timing reduction of bench.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2203_11733_b200.shard import balanced_row_split, row_work


@pytest.mark.parametrize("n,world", [(1, 1), (7, 2), (100, 3), (1344, 8), (11340, 8), (200000, 8)])
def test_balanced_split_tiles_and_balances(n, world):
    parts = balanced_row_split(n, world)
    assert parts[0][0] == 0 and parts[-1][1] == n
    assert all(a <= b for a, b in parts)
    assert all(parts[k][1] == parts[k + 1][0] for k in range(world - 1))
    work = [row_work(n, a, b) for a, b in parts]
    assert sum(work) == n * (n + 1) // 2
    if n >= 100 * world:
        assert max(work) <= 1.01 * (sum(work) / world)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, P, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle_lib as O
    n = len(P)
    a, b = balanced_row_split(n, world)[rank]
    # this rank's rows of the upper triangle (CPU oracle in place of the rank's GPU)
    block = np.zeros((n, n))
    for i in range(a, b):
        js = np.arange(i, n)
        u, _, st = O.u_pairs("orc", np.repeat(P[i:i + 1], len(js), axis=0), P[js], nthreads=1)
        area_i = (P[i, 3] - P[i, 2]) * (P[i, 5] - P[i, 4])
        area_j = (P[js, 3] - P[js, 2]) * (P[js, 5] - P[js, 4])
        block[i, js] = u / (area_i * area_j)
    t = torch.from_numpy(block)
    gathered = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    # bench.py reduces per-rank step times with MAX
    ms = torch.tensor([10.0 + rank])
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        full = sum(g.numpy() for g in gathered)
        full = np.triu(full) + np.triu(full, 1).T
        np.save(out_path, full)
        assert ms.item() == 10.0 + world - 1
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_row_blocks_reassemble(tmp_path):
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    import oracle_lib as O
    from test_gpu_assembly import two_boxes
    P, _ = two_boxes(0.1)
    out = str(tmp_path / "full.npy")
    mp.spawn(_worker, args=(2, _free_port(), P, out), nprocs=2, join=True)
    full = np.load(out)
    ref, conv, rc = O.assemble("orc", P, nthreads=4)
    assert rc == 0
    assert np.array_equal(full, ref)
