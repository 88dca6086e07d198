"""TEST INFRASTRUCTURE: a torch restatement of the device recurrence of
gbem_pcg_extract_cmatrix_dev (csrc/gbem_pcg.cu) — K simultaneous block-Jacobi
preconditioned CG recurrences on row blocks, with the same per-column freeze
rule (alpha = beta = 0 once ||r|| / ||b|| <= tol) — driven by torch.distributed
collectives so the sharded algorithm runs under gloo on CPU ranks
(tests/test_distributed.py) and pins the GPU run's iteration counts."""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

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


