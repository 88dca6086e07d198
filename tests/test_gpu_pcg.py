"""Sharded-solver building blocks on the GPU (paper_2203_11733_b200/pcg.py):
full-row assembly, the row-block product, the kept factor, and the block-Jacobi
PCG C-matrix against the direct Cholesky extraction."""
import ctypes as C

import numpy as np
import pytest
import torch

import paper_2203_11733_b200 as g
from paper_2203_11733_b200._native import PanelArrays
from paper_2203_11733_b200.pcg import GpuRowBlockOps, sharded_cmatrix
from paper_2203_11733_b200.shard import panels_to_device
from test_gpu_assembly import two_boxes

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rows,n,K,ldp", [(1, 1, 1, 1), (37, 300, 5, 5), (128, 1000, 8, 8), (250, 777, 13, 16),
                                           (129, 515, 40, 40), (300, 1000, 64, 64), (70, 333, 70, 72), (5, 17, 9, 9)])
def test_rowblock_matvec(ctx, rows, n, K, ldp):
    gen = torch.Generator(device="cpu").manual_seed(rows + n)
    ld = ((n + 7) // 8) * 8
    A = torch.randn((rows, ld), generator=gen, dtype=torch.float64).cuda()
    P = torch.randn((n, ldp), generator=gen, dtype=torch.float64).cuda()
    Q = torch.full((rows, K), float("nan"), dtype=torch.float64, device="cuda")
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    ctx.check(ctx.lib.gbem_rowblock_matvec_dev(ctx.h, C.c_void_p(A.data_ptr()), ld, rows, n,
                                               C.c_void_p(P.data_ptr()), ldp, K, C.c_void_p(Q.data_ptr()), K))
    ref = A[:, :n].cpu().numpy() @ P[:, :K].cpu().numpy()
    Qh = Q.cpu().numpy()
    assert np.all(np.abs(Qh - ref) <= 1e-13 * np.abs(ref) + 1e-12 * np.abs(ref).max())


def test_full_rows_match_symmetric_assembly(ctx):
    P, _ = two_boxes(0.05)
    n = len(P)
    A, _ = ctx.assemble_single(PanelArrays.from_matrix(P))
    pd = panels_to_device(PanelArrays.from_matrix(P), torch.device("cuda", 0))
    ops = GpuRowBlockOps(ctx, pd, n, 1, 3)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    blk = ops.assemble(with_stats=True)[:, :n].cpu().numpy()
    ref = A[ops.row_begin:ops.row_end]
    rel = np.abs(blk - ref) / np.abs(ref)
    assert rel.max() <= 1e-13, rel.max()
    assert ops.astats.pairs_total == ops.rows * n
    # the upper triangle is the same computation as the symmetric path
    iu = np.triu_indices(ops.rows, ops.row_begin, n)
    assert np.array_equal(blk[iu], ref[iu])


def test_factor_then_repeated_solves(ctx):
    rng = np.random.default_rng(3)
    m, ld = 300, 320
    G = rng.standard_normal((m, m))
    S = G @ G.T + m * np.eye(m)
    M = torch.zeros((m, ld), dtype=torch.float64)
    M[:, :m] = torch.from_numpy(S)
    M = M.cuda()
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    ctx.check(ctx.lib.gbem_spd_factor_dev(ctx.h, C.c_void_p(M.data_ptr()), m, ld, None))
    for k in (1, 3, 40):
        B = rng.standard_normal((k, m))
        dB = torch.from_numpy(B).cuda()
        dX = torch.empty_like(dB)
        res = torch.empty(k, dtype=torch.float64, device="cuda")
        ctx.check(ctx.lib.gbem_spd_solve_factored_dev(ctx.h, C.c_void_p(dB.data_ptr()), k, C.c_void_p(dX.data_ptr()),
                                                      C.c_void_p(res.data_ptr()), None))
        X = dX.cpu().numpy()
        ref = np.linalg.solve(S, B.T).T
        assert np.abs(X - ref).max() <= 1e-12 * np.abs(ref).max()
        assert res.max().item() <= 1e-13


def test_non_spd_block_reports_pivot(ctx):
    m = 130
    M = torch.eye(m, dtype=torch.float64, device="cuda")
    M[129, 129] = -1.0
    rc = ctx.lib.gbem_spd_factor_dev(ctx.h, C.c_void_p(M.data_ptr()), m, m, None)
    assert rc == 2
    assert "not positive definite" in ctx.lib.gbem_last_error(ctx.h).decode()


@pytest.mark.parametrize("sub_blocks", [1, 5])
def test_pcg_cmatrix_matches_direct(ctx, sub_blocks):
    m = g.config_model(1, seed=1, scale=0.5)
    ps = m.partition(1)
    ids = m.net_ids
    col = {nid: k for k, nid in enumerate(ids)}
    net = np.array([col.get(int(v), -1) if k == 0 else -1 for v, k in zip(ps.net, ps.kind)], dtype=np.int32)
    K, eps = len(ids), m.info()["eps_r"]
    Cd, _, _, _ = ctx.extract_cmatrix(ps.arrays(), net, K, eps)
    Cp, res = sharded_cmatrix(ctx, ps.arrays(), net, K, eps, tol=1e-12, sub_blocks=sub_blocks)
    assert res.converged, res.rel_resid
    if sub_blocks == 1:
        assert res.iterations <= 2      # one Jacobi block = the exact inverse
    else:
        assert res.iterations > 2
    assert np.abs(Cp - Cd).max() <= 1e-9 * np.abs(Cd).max(), np.abs(Cp - Cd).max() / np.abs(Cd).max()


def test_async_mode_defers_pivot_check(ctx):
    """gbem_ctx_set_async: the factor returns immediately and the non-SPD pivot is
    reported by gbem_ctx_sync with the synchronous call's message."""
    m = 130
    M = torch.eye(m, dtype=torch.float64, device="cuda")
    M[129, 129] = -1.0
    ctx.set_stream(0)
    ctx.check(ctx.lib.gbem_ctx_set_async(ctx.h, 1))
    try:
        assert ctx.lib.gbem_spd_factor_dev(ctx.h, C.c_void_p(M.data_ptr()), m, m, None) == 0
        rc = ctx.lib.gbem_ctx_sync(ctx.h)
        assert rc == 2
        assert "pivot at row 129" in ctx.lib.gbem_last_error(ctx.h).decode()
        assert ctx.lib.gbem_ctx_sync(ctx.h) == 0  # reported once
    finally:
        ctx.check(ctx.lib.gbem_ctx_set_async(ctx.h, 0))
