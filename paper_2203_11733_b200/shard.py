"""Row-block sharding of the Galerkin assembly across ranks (one process per GPU).

Assembly needs no communication (every entry is an independent pure function of
two panels): rank r owns a contiguous row range of the upper
triangle, balanced by unique-pair work, not by row count.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np


def row_work(n: int, a: int, b: int) -> int:
    """Unique pairs (i, j >= i) with row i in [a, b)."""
    return (b - a) * n - (b * (b - 1) - a * (a - 1)) // 2


def balanced_row_split(n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous row ranges with equal upper-triangle work n(n+1)/2 / world.

    W(b) = sum_{i<b} (n - i) = b n - b(b-1)/2; boundary b_r solves
    W(b) = r T / world (T = n(n+1)/2), rounded to the nearest row.
    """
    if world < 1:
        raise ValueError("world must be >= 1")
    total = n * (n + 1) // 2
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        # b^2 - (2n+1) b + 2 target = 0, smaller root
        disc = (2 * n + 1) ** 2 - 8 * target
        b = int(round(((2 * n + 1) - math.sqrt(max(disc, 0.0))) / 2))
        bounds.append(min(max(b, bounds[-1]), n))
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


class ShardedAssembler:
    """This rank's row block of the assembled matrix, on its own GPU.

    block[i - row_begin, j] = A[i, j] for j >= i (entries j < i are not written).
    """

    def __init__(self, ctx, panels_dev: dict, n: int, rank: int, world: int, cfg=None):
        import torch
        from . import _native as N
        self.ctx, self.n, self.rank, self.world = ctx, n, rank, world
        self.row_begin, self.row_end = balanced_row_split(n, world)[rank]
        self.ld = ((n + 7) // 8) * 8
        dev = panels_dev["level"].device
        self.block = torch.zeros((max(self.row_end - self.row_begin, 1), self.ld), dtype=torch.float64, device=dev)
        dp = C.POINTER(C.c_double)
        self._keep = panels_dev
        self.panels = N.GbemPanels(
            C.cast(C.c_void_p(panels_dev["axis"].data_ptr()), C.POINTER(C.c_uint8)),
            *[C.cast(C.c_void_p(panels_dev[k].data_ptr()), dp) for k in ("level", "a0", "a1", "b0", "b1")])
        self.cfg = cfg or ctx.quad()
        self.stats = N.GbemAssemblyStats()

    def assemble(self, with_stats: bool = False):
        rc = self.ctx.lib.gbem_assemble_rows_dev(self.ctx.h, C.byref(self.panels), self.n, self.row_begin,
                                                 self.row_end, C.byref(self.cfg), C.c_void_p(self.block.data_ptr()),
                                                 self.ld, C.byref(self.stats) if with_stats else None)
        self.ctx.check(rc)
        return self.block

    @property
    def unique_pairs(self) -> int:
        return row_work(self.n, self.row_begin, self.row_end)


def panels_to_device(ps, device) -> dict:
    import torch
    return {k: torch.from_numpy(np.ascontiguousarray(v)).to(device) for k, v in
            dict(axis=ps.axis.astype(np.uint8), level=ps.level, a0=ps.a0, a1=ps.a1, b0=ps.b0, b1=ps.b1).items()}
