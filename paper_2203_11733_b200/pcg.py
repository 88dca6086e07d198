"""Row-block sharded block-Jacobi PCG for the single-layer Galerkin system.

SURVEY.md §8e: when A does not fit one GPU (config 4: 80 GB; config 5: 320 GB)
the system A X = B (B = one indicator column per net, extraction.hpp:118-130)
is solved with preconditioned conjugate gradients over row blocks.  Rank r owns
rows [a_r, b_r) of A in full (every j; mirrored entries are recomputed locally
by ``gbem_assemble_rows_full_dev``, no communication), and the preconditioner is
the Cholesky factor of its own diagonal block A[a_r:b_r, a_r:b_r] (the DMMA
factorisation of the direct path, ``gbem_spd_factor_dev``).  Per iteration:

* ``all_gather`` of the search directions P (n x K; NCCL over NVLink),
* the local product Q_r = A_r P (``gbem_rowblock_matvec_dev``, HBM-bound on A_r),
* ``all_reduce`` of 2K (then 2K) column inner products,
* the block-Jacobi solve Z_r = A_rr^-1 R_r (``gbem_spd_solve_factored_dev``).

The K columns run as K independent CG recurrences sharing every kernel launch
and collective.  The reference has no iterative solver (solver.hpp:24 is dense
Cholesky only); the result is checked against the direct path
(tests/test_gpu_pcg.py) and against numpy on CPU ranks (tests/test_distributed.py).

Rows are split evenly (ceil(n / world) per rank): the full-row assembly and the
product A_r P both cost rows x n, so equal rows are equal work, and equal
blocks let the gather run as one fixed-size ``all_gather_into_tensor``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

EPS0 = 8.854187817e-12  # extraction.hpp:55 (F/m)


def equal_row_split(n: int, world: int) -> list[tuple[int, int]]:
    """Row ranges of ceil(n / world) rows (the last ones may be shorter or empty)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    m = -(-n // world) if n else 0
    return [(min(r * m, n), min((r + 1) * m, n)) for r in range(world)]


class Comm:
    """The two collectives the PCG needs, over a torch.distributed group
    (NCCL on GPUs, gloo in the CPU tests); identity at world size 1."""

    def __init__(self, group=None):
        self.group = group
        self.on = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if self.on else 1
        self.rank = dist.get_rank(group) if self.on else 0

    def all_gather_rows(self, local: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        """local: (m, K) with m = ceil(n / world); out: (world * m, K)."""
        if self.world == 1:
            out.copy_(local)
        else:
            dist.all_gather_into_tensor(out, local.contiguous(), group=self.group)
        return out

    def all_reduce(self, t: torch.Tensor) -> torch.Tensor:
        if self.world > 1:
            dist.all_reduce(t, group=self.group)
        return t


@dataclass
class PcgResult:
    x: torch.Tensor               # (rows, K) this rank's rows of X
    iterations: int
    rel_resid: np.ndarray         # (K,) ||b - A x|| / ||b|| from the recurrence
    converged: bool
    history: list = field(default_factory=list)


def block_jacobi_pcg(ops, b: torch.Tensor, comm: Comm, tol: float = 1e-12, max_iter: int = 1000,
                     keep_history: bool = False) -> PcgResult:
    """K simultaneous preconditioned CG recurrences on the sharded system.

    ops.matvec(P_full) -> A_r P (rows, K); ops.precond(R) -> A_rr^-1 R (rows, K);
    ops.m = ceil(n / world) (rows of the gather slot).  b: (rows, K) local rows.
    A column stops updating once its relative residual is <= tol.
    """
    rows, K = b.shape
    dev, dt = b.device, b.dtype
    m = ops.m
    x = torch.zeros_like(b)
    r = b.clone()
    z = ops.precond(r)
    p = z.clone()
    slot = torch.zeros((m, K), dtype=dt, device=dev)
    p_full = torch.zeros((comm.world * m, K), dtype=dt, device=dev)
    red = torch.stack([(r * z).sum(0), (b * b).sum(0)])
    comm.all_reduce(red)
    rz, bb = red[0].clone(), red[1].clone()
    bnorm = torch.sqrt(bb).clamp_min(torch.finfo(dt).tiny)
    active = torch.ones(K, dtype=torch.bool, device=dev)
    rel = torch.ones(K, dtype=dt, device=dev)
    hist = []
    it = 0
    for it in range(1, max_iter + 1):
        slot[:rows] = p
        comm.all_gather_rows(slot, p_full)
        q = ops.matvec(p_full)
        pq = (p * q).sum(0)
        comm.all_reduce(pq)
        alpha = torch.where(active & (pq > 0), rz / torch.where(pq > 0, pq, torch.ones_like(pq)),
                            torch.zeros_like(pq))
        x += alpha * p
        r -= alpha * q
        z = ops.precond(r)
        red = torch.stack([(r * r).sum(0), (r * z).sum(0)])
        comm.all_reduce(red)
        rel = torch.sqrt(red[0]) / bnorm
        if keep_history:
            hist.append(rel.max().item())
        active = active & (rel > tol)
        if not bool(active.any()):
            break
        beta = torch.where(active, red[1] / torch.where(rz != 0, rz, torch.ones_like(rz)), torch.zeros_like(rz))
        rz = torch.where(active, red[1], rz)
        p = torch.where(active, z + beta * p, p)
    relh = rel.cpu().numpy()
    return PcgResult(x, it, relh, bool((relh <= tol).all()), hist)


class GpuRowBlockOps:
    """This rank's full rows of A on its GPU, the factored diagonal block, and the
    matvec / preconditioner of block_jacobi_pcg, all through the C-ABI.

    ``sub_blocks`` > 1 splits the rank's diagonal block into that many Jacobi
    blocks (one context each), which exercises the multi-block recurrence on a
    single GPU.
    """

    def __init__(self, ctx, panels_dev: dict, n: int, rank: int, world: int, cfg=None, sub_blocks: int = 1):
        from . import _native as N
        self.N = N
        self.ctx, self.n = ctx, n
        self.row_begin, self.row_end = equal_row_split(n, world)[rank]
        self.rows = self.row_end - self.row_begin
        self.m = -(-n // world)
        self.ld = ((n + 7) // 8) * 8
        dev = panels_dev["level"].device
        self.dev = dev
        self.block = torch.zeros((max(self.rows, 1), self.ld), dtype=torch.float64, device=dev)
        dp = C.POINTER(C.c_double)
        self._keep = panels_dev
        self.panels = N.GbemPanels(
            C.cast(C.c_void_p(panels_dev["axis"].data_ptr()), C.POINTER(C.c_uint8)),
            *[C.cast(C.c_void_p(panels_dev[k].data_ptr()), dp) for k in ("level", "a0", "a1", "b0", "b1")])
        self.cfg = cfg or ctx.quad()
        self.astats = N.GbemAssemblyStats()
        # Jacobi blocks inside this rank's rows
        nb = max(1, min(sub_blocks, self.rows or 1))
        cuts = [self.rows * k // nb for k in range(nb + 1)]
        self.jblocks = [(cuts[k], cuts[k + 1]) for k in range(nb) if cuts[k + 1] > cuts[k]]
        stream = torch.cuda.current_stream(dev).cuda_stream
        self.pctx = [ctx] + [N.Context(dev.index) for _ in self.jblocks[1:]]
        for c in self.pctx[1:]:
            c.set_stream(stream)

    def assemble(self, with_stats: bool = False):
        rc = self.ctx.lib.gbem_assemble_rows_full_dev(
            self.ctx.h, C.byref(self.panels), self.n, self.row_begin, self.row_end, C.byref(self.cfg),
            C.c_void_p(self.block.data_ptr()), self.ld, C.byref(self.astats) if with_stats else None)
        self.ctx.check(rc)
        return self.block

    def factor(self):
        base = self.block.data_ptr()
        for c, (a, b) in zip(self.pctx, self.jblocks):
            ptr = base + 8 * (a * self.ld + self.row_begin + a)
            c.check(c.lib.gbem_spd_factor_dev(c.h, C.c_void_p(ptr), b - a, self.ld, None))

    def matvec(self, p_full: torch.Tensor) -> torch.Tensor:
        K = p_full.shape[1]
        q = torch.empty((self.rows, K), dtype=torch.float64, device=self.dev)
        if self.rows:
            rc = self.ctx.lib.gbem_rowblock_matvec_dev(self.ctx.h, C.c_void_p(self.block.data_ptr()), self.ld,
                                                       self.rows, self.n, C.c_void_p(p_full.data_ptr()), K,
                                                       K, C.c_void_p(q.data_ptr()), K)
            self.ctx.check(rc)
        return q

    def precond(self, r: torch.Tensor) -> torch.Tensor:
        K = r.shape[1]
        z = torch.empty_like(r)
        for c, (a, b) in zip(self.pctx, self.jblocks):
            rt = r[a:b].t().contiguous()     # (K, m): column-major m x K
            zt = torch.empty_like(rt)
            c.check(c.lib.gbem_spd_solve_factored_dev(c.h, C.c_void_p(rt.data_ptr()), K, C.c_void_p(zt.data_ptr()),
                                                      None, None))
            z[a:b] = zt.t()
        return z


def sharded_cmatrix(ctx, P, net_of_panel: np.ndarray, K: int, eps_r: float, cfg=None, group=None,
                    tol: float = 1e-12, max_iter: int = 1000, sub_blocks: int = 1):
    """C-matrix extraction on row-block shards (every rank of ``group`` calls it
    with the same panels).  P: ``_native.PanelArrays``.  Returns (C (K, K) numpy,
    PcgResult); C is identical on every rank."""
    from .shard import panels_to_device
    comm = Comm(group)
    dev = torch.device("cuda", torch.cuda.current_device())
    ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    pd = panels_to_device(P, dev)
    ops = GpuRowBlockOps(ctx, pd, P.n, comm.rank, comm.world, cfg, sub_blocks)
    ops.assemble()
    ops.factor()
    net = torch.from_numpy(np.ascontiguousarray(net_of_panel, dtype=np.int32)).to(dev)
    net_local = net[ops.row_begin:ops.row_end].contiguous()
    cols = torch.arange(K, device=dev, dtype=torch.int32)
    b = (net_local[:, None] == cols[None, :]).to(torch.float64)
    res = block_jacobi_pcg(ops, b, comm, tol=tol, max_iter=max_iter)
    # partial net charges of the local rows (k_net_charges), then summed over ranks
    Cm = torch.zeros(K * K, dtype=torch.float64, device=dev)
    if ops.rows:
        xt = res.x.t().contiguous()          # (K, rows)
        ctx.check(ctx.lib.gbem_net_charges_dev(ctx.h, C.c_void_p(net_local.data_ptr()), ops.rows,
                                               C.c_void_p(xt.data_ptr()), K, K, eps_r * EPS0 * 1e-6,
                                               C.c_void_p(Cm.data_ptr()), None))
    comm.all_reduce(Cm)
    return Cm.view(K, K).cpu().numpy(), res
