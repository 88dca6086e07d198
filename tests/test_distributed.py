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


# --- sharded block-Jacobi PCG (paper_2203_11733_b200/pcg.py) -------------------------

from paper_2203_11733_b200.pcg import equal_row_split  # noqa: E402
from pcg_restatement import Comm, block_jacobi_pcg  # noqa: E402


@pytest.mark.parametrize("n,world", [(0, 2), (1, 2), (7, 2), (10, 3), (1344, 8), (100000, 8)])
def test_equal_row_split(n, world):
    parts = equal_row_split(n, world)
    assert len(parts) == world and parts[0][0] == 0 and parts[-1][1] == n
    assert all(parts[k][1] == parts[k + 1][0] for k in range(world - 1))
    m = -(-n // world) if n else 0
    assert all(0 <= b - a <= m for a, b in parts)


class _CpuRowBlockOps:
    """Test stand-in for GpuRowBlockOps: the same row block and Jacobi block on CPU
    torch tensors, so the recurrence and its collectives run under gloo."""

    def __init__(self, A, rank, world):
        n = A.shape[0]
        self.row_begin, self.row_end = equal_row_split(n, world)[rank]
        self.rows = self.row_end - self.row_begin
        self.m = -(-n // world)
        self.n = n
        self.block = torch.from_numpy(A[self.row_begin:self.row_end].copy())
        self.L = torch.linalg.cholesky(self.block[:, self.row_begin:self.row_end])

    def matvec(self, p_full):
        return self.block @ p_full[:self.n]

    def precond(self, r):
        return torch.cholesky_solve(r, self.L)


def _pcg_worker(rank, world, port, A, B, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = Comm()
    ops = _CpuRowBlockOps(A, rank, world)
    b = torch.from_numpy(B[ops.row_begin:ops.row_end].copy())
    res = block_jacobi_pcg(ops, b, comm, tol=1e-13, max_iter=500)
    xs = [torch.zeros((ops.m, B.shape[1]), dtype=torch.float64) for _ in range(world)]
    slot = torch.zeros((ops.m, B.shape[1]), dtype=torch.float64)
    slot[:ops.rows] = res.x
    dist.all_gather(xs, slot)
    if rank == 0:
        X = torch.cat(xs)[:A.shape[0]].numpy()
        np.save(out_path, X)
        assert res.converged, res.rel_resid
        assert res.iterations > 1
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_pcg_matches_direct_solve(tmp_path, world):
    """Single-layer Galerkin matrix (CPU oracle assembly) with one indicator
    right-hand side per box: the sharded recurrence under gloo reaches the
    dense solution."""
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    import oracle_lib as O
    from test_gpu_assembly import two_boxes
    P, n1 = two_boxes(0.1)
    A, conv, rc = O.assemble("orc", P, nthreads=4)
    assert rc == 0
    n = len(P)
    B = np.zeros((n, 2))
    B[:n1, 0] = 1.0
    B[n1:, 1] = 1.0
    out = str(tmp_path / "x.npy")
    mp.spawn(_pcg_worker, args=(world, _free_port(), A, B, out), nprocs=world, join=True)
    X = np.load(out)
    Xd = np.linalg.solve(A, B)
    assert np.abs(X - Xd).max() <= 1e-9 * np.abs(Xd).max()
    # capacitance-style column sums agree to the solve tolerance
    np.testing.assert_allclose(X.sum(0), Xd.sum(0), rtol=1e-11)


# --- host collectives plugged into the C-ABI (paper_2203_11733_b200/pcg.py) ------------

def _coll_worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2203_11733_b200.pcg import HostCollectives
    hc = HostCollectives(device=False)
    # the library calls the C function pointers; call them the same way
    send = np.arange(5, dtype=np.float64) + 10 * rank
    recv = np.zeros(5 * world)
    assert hc.struct.all_gather(None, send.ctypes.data, recv.ctypes.data, 5, None) == 0
    buf = np.full(3, rank + 1.0)
    assert hc.struct.all_reduce_sum(None, buf.ctypes.data, 3, None) == 0
    if rank == 0:
        np.savez(out_path, recv=recv, buf=buf)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_host_collectives_callbacks(tmp_path, world):
    out = str(tmp_path / "c.npz")
    mp.spawn(_coll_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    d = np.load(out)
    assert np.array_equal(d["recv"], np.concatenate([np.arange(5) + 10 * r for r in range(world)]))
    assert np.array_equal(d["buf"], np.full(3, world * (world + 1) / 2))
