"""GPU assembly + SPD solve parity against the CPU oracle on identical panel lists."""
import numpy as np
import pytest

import oracle_lib as O
from paper_2203_11733_b200._native import PanelArrays

pytestmark = pytest.mark.gpu


def box_panels(lo, hi, h):
    """Uniform panels of edge ~h on the 6 faces of a box (row order: face by face)."""
    rows = []
    for axis in range(3):
        i0, i1 = {0: (1, 2), 1: (0, 2), 2: (0, 1)}[axis]
        na = max(1, int(round((hi[i0] - lo[i0]) / h)))
        nb = max(1, int(round((hi[i1] - lo[i1]) / h)))
        ea = np.linspace(lo[i0], hi[i0], na + 1)
        eb = np.linspace(lo[i1], hi[i1], nb + 1)
        for lvl in (lo[axis], hi[axis]):
            for ia in range(na):
                for ib in range(nb):
                    rows.append([axis, lvl, ea[ia], ea[ia + 1], eb[ib], eb[ib + 1]])
    return np.array(rows)


def two_boxes(h):
    a = box_panels((-0.5, -0.15, -0.05), (0.5, -0.05, 0.05), h)
    b = box_panels((-0.5, 0.05, -0.05), (0.5, 0.15, 0.05), h)
    return np.vstack([a, b]), len(a)


def test_assembly_matches_oracle(ctx):
    P, n1 = two_boxes(0.05)
    A_gpu, st = ctx.assemble_single(PanelArrays.from_matrix(P))
    A_ref, conv, rc = O.assemble("orc", P, nthreads=16)
    assert rc == 0 and conv
    assert st.pairs_total == len(P) * (len(P) + 1) // 2
    assert st.pairs_coplanar + st.pairs_parallel + st.pairs_orthogonal + st.pairs_far == st.pairs_total
    assert np.array_equal(A_gpu, A_gpu.T)
    rel = np.abs(A_gpu - A_ref) / np.abs(A_ref)
    # far entries: the reference value itself is only good to its cancellation floor;
    # compare those against the composite-Gauss truth instead
    iu = np.triu_indices(len(P))
    g = O.gap_ratio(P[iu[0]], P[iu[1]])
    near = g < 1.5
    assert rel[iu][near].max() <= 1e-10, rel[iu][near].max()
    far_idx = np.flatnonzero(~near)
    sel = far_idx[:: max(1, len(far_idx) // 2000)]
    ii, jj = iu[0][sel], iu[1][sel]
    truth = O.truth_pairs(P[ii], P[jj]) / ((P[ii, 3] - P[ii, 2]) * (P[ii, 5] - P[ii, 4]) * (P[jj, 3] - P[jj, 2]) * (P[jj, 5] - P[jj, 4]))
    relt = np.abs(A_gpu[ii, jj] - truth) / truth
    assert relt.max() <= 1e-10, relt.max()
    lim = np.maximum(1e-10 * np.abs(A_ref[ii, jj]), 2 * np.abs(A_ref[ii, jj] - truth))
    assert np.all(np.abs(A_gpu[ii, jj] - A_ref[ii, jj]) <= lim + 1e-13 * truth)


@pytest.mark.parametrize("n", [1, 7, 128, 129, 300, 1000])
def test_cholesky_random_spd(ctx, n):
    rng = np.random.default_rng(n)
    M = rng.normal(size=(n, n))
    A = M.T @ M + n * np.eye(n)
    B = rng.normal(size=(n, 3))
    ctx.matrix_upload(A)
    X, res, st = ctx.spd_solve(B)
    Xn = np.linalg.solve(A, B)
    assert np.abs(X - Xn).max() <= 1e-10 * np.abs(Xn).max()
    assert res.max() <= 1e-12
    assert np.allclose(res, np.linalg.norm(A @ X - B, axis=0) / np.linalg.norm(B, axis=0), rtol=1e-2, atol=2e-15)


def test_cholesky_rejects_indefinite(ctx):
    from paper_2203_11733_b200._native import GbemError
    A = np.array([[1.0, 2.0], [2.0, 1.0]])  # test_solver.cpp:82-90
    ctx.matrix_upload(A)
    with pytest.raises(GbemError) as ei:
        ctx.spd_solve(np.ones(2))
    assert ei.value.code == 2
    assert "matrix not positive definite" in str(ei.value)
    assert "row 1" in str(ei.value)


def test_assembled_system_solve(ctx):
    P, n1 = two_boxes(0.05)
    A_gpu, _ = ctx.assemble_single(PanelArrays.from_matrix(P))
    B = np.zeros((len(P), 2))
    B[:n1, 0] = 1.0
    B[n1:, 1] = 1.0
    X, res, st = ctx.spd_solve(B)
    Xn = np.linalg.solve(A_gpu, B)
    assert np.abs(X - Xn).max() <= 1e-9 * np.abs(Xn).max()
    assert res.max() <= 1e-10


def test_row_block_sharded_assembly_matches_full(ctx):
    """gbem_assemble_rows_dev: rank blocks (simulated sequentially on one GPU) equal
    the rows of the full assembly bit for bit (no communication needed)."""
    import torch
    from paper_2203_11733_b200.shard import ShardedAssembler, panels_to_device
    P, _ = two_boxes(0.05)
    A_full, _ = ctx.assemble_single(PanelArrays.from_matrix(P))
    import paper_2203_11733_b200.api as api
    dev = torch.device("cuda", 0)
    cols = dict(axis=P[:, 0].astype(np.uint8), level=P[:, 1], a0=P[:, 2], a1=P[:, 3], b0=P[:, 4], b1=P[:, 5])
    pdev = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in cols.items()}
    n = len(P)
    world = 3
    for rank in range(world):
        sh = ShardedAssembler(ctx, pdev, n, rank, world)
        blk = sh.assemble(with_stats=True).cpu().numpy()
        assert sh.stats.pairs_total == sh.unique_pairs
        for i in range(sh.row_begin, sh.row_end):
            assert np.array_equal(blk[i - sh.row_begin, i:n], A_full[i, i:n])


@pytest.mark.parametrize("nrhs", [1, 2, 3, 4, 5, 6, 7, 8, 16])
def test_cholesky_ragged_after_nan_shared(ctx, nrhs):
    """every solve path initialises the shared memory it
    reads.  NaN is left in every SM's shared memory by a prior kernel, then a
    ragged system (n % 128 != 0) is solved at each right-hand-side width."""
    n = 2832
    rng = np.random.default_rng(nrhs)
    M = rng.normal(size=(n, n)) / np.sqrt(n)
    A = M.T @ M + 2.0 * np.eye(n)
    B = rng.normal(size=(n, nrhs))
    ctx.matrix_upload(A)
    ctx.fill_shared(float("nan"))
    X, res, st = ctx.spd_solve(B)
    assert np.isfinite(X).all()
    Xn = np.linalg.solve(A, B)
    assert np.abs(X - Xn).max() <= 1e-10 * np.abs(Xn).max()
    assert res.max() <= 1e-12


def test_cholesky_many_rhs(ctx):
    """nrhs > 64: the solve loops over right-hand-side chunks."""
    n = 700
    rng = np.random.default_rng(70)
    M = rng.normal(size=(n, n)) / np.sqrt(n)
    A = M.T @ M + np.eye(n)
    B = rng.normal(size=(n, 100))
    ctx.matrix_upload(A)
    X, res, st = ctx.spd_solve(B)
    Xn = np.linalg.solve(A, B)
    assert np.abs(X - Xn).max() <= 1e-10 * np.abs(Xn).max()
    assert res.max() <= 1e-12


@pytest.mark.parametrize("n,nrhs", [(3000, 5), (3000, 17), (16400, 17), (16400, 40)])
def test_matrix_apply_matches_numpy(ctx, n, nrhs):
    """gbem_matrix_apply_dev: Y = A X from the preserved upper triangle + saved
    diagonal (the residual product of solver.hpp:47): the scalar kernel below
    n = 16,384, the DMMA k_symm_dmma above (32 right-hand sides per pass);
    the same before and after the factorisation overwrites the lower triangle."""
    import torch
    rng = np.random.default_rng(n + nrhs)
    M = rng.standard_normal((n, 48)) / 7
    A = M @ M.T + 4.0 * np.eye(n)
    X = rng.standard_normal((nrhs, n))  # column-major n x nrhs = row-major (nrhs, n)
    ctx.matrix_upload(A)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    dX = torch.from_numpy(X).cuda()
    dY = torch.full_like(dX, float("nan"))
    import ctypes as C
    ctx.check(ctx.lib.gbem_matrix_apply_dev(ctx.h, C.c_void_p(dX.data_ptr()), nrhs, C.c_void_p(dY.data_ptr())))
    ref = X @ A  # rows: (A x_q)^T, A symmetric
    Y1 = dY.cpu().numpy()
    scale = np.abs(A).sum(1).max() * np.abs(X).max()
    assert np.abs(Y1 - ref).max() <= 1e-13 * scale
    ctx.spd_solve(rng.standard_normal((n, 2)))  # factor: the lower triangle now holds L
    dY.fill_(float("nan"))
    ctx.check(ctx.lib.gbem_matrix_apply_dev(ctx.h, C.c_void_p(dX.data_ptr()), nrhs, C.c_void_p(dY.data_ptr())))
    # (the scalar kernel folds column chunks with atomics: same values up to summation order)
    assert np.abs(dY.cpu().numpy() - ref).max() <= 1e-13 * scale
    ctx.set_stream(0)


def test_concurrent_assembly_bit_identical_to_serial(ctx, monkeypatch):
    """Without per-phase timing (stats = NULL) an assembly runs its near-field kernels on a second
    stream, deals the far-field kernels over four, classifies chunk t + 1 while chunk t is evaluated
    and defers the near-contact (Romberg-route) pairs to one launch at its end; with stats the phases
    run one after the other.  Both must give the same matrix bit for bit — on the 2,880-panel
    near-contact set (every near route, 240 Romberg pairs) cut into ~60 chunks by a small queue."""
    import json
    import pathlib
    import torch
    from paper_2203_11733_b200.shard import ShardedAssembler
    g = json.load(open(pathlib.Path(__file__).parent / "golden" / "near_contact_golden.json"))
    A, B = np.array(g["A"]), np.array(g["B"])
    P = np.empty((2 * len(A), 6))
    P[0::2] = A
    P[1::2] = B
    dev = torch.device("cuda", 0)
    cols = dict(axis=P[:, 0].astype(np.uint8), level=P[:, 1], a0=P[:, 2], a1=P[:, 3], b0=P[:, 4], b1=P[:, 5])
    pdev = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in cols.items()}
    n = len(P)
    results = {}
    for cap in (None, 1 << 16):
        if cap is None:
            monkeypatch.delenv("GBEM_QUEUE_CAP", raising=False)
        else:
            monkeypatch.setenv("GBEM_QUEUE_CAP", str(cap))
        for with_stats in (True, False):
            sh = ShardedAssembler(ctx, pdev, n, 0, 1)
            results[(cap, with_stats)] = sh.assemble(with_stats=with_stats).clone()
            if with_stats:
                assert sh.stats.pairs_total == n * (n + 1) // 2
                assert sh.stats.pairs_near_romberg > 100
    torch.cuda.synchronize()
    ref = results[(None, True)]
    for key, blk in results.items():
        assert torch.equal(blk, ref), key
