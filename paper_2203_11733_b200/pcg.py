"""Row-block sharded C-matrix extraction: the host side of
``gbem_pcg_extract_cmatrix_dev`` (include/gbem_gpu.h, csrc/gbem_pcg.cu).

SURVEY.md §8e: when A does not fit one GPU (config 4: 74 GB; config 5: 320 GB)
the system A X = B (B = one indicator column per net, extraction.hpp:118-130)
is solved by block-Jacobi preconditioned conjugate gradients over row blocks.
Rank r owns rows [r m, min((r+1) m, n)), m = ceil(n / world), of A in full
(assembled locally, no communication), the preconditioner is the explicit
inverse of its diagonal block(s), and every iteration is one all-gather of the
search directions plus two all-reduces of K-vectors — all enqueued by the
library on the context's stream (NCCL owned by the context, or the host's own
collectives plugged in through ``gbem_collectives``).  The reference has no
iterative solver (solver.hpp:24 is dense Cholesky only); the result is checked
against the direct path (tests/test_gpu_pcg.py) and the recurrence against a
CPU restatement under gloo (tests/test_distributed.py).

This module only wires a ``torch.distributed`` group to the context:
``attach`` picks NCCL (the unique id travels over the group) or host-staged
collectives for any other backend (gloo in the multi-process tests).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N

EPS0 = 8.854187817e-12  # extraction.hpp:20 (F/m)


def equal_row_split(n: int, world: int) -> list[tuple[int, int]]:
    """Row ranges of ceil(n / world) rows (the last ones may be shorter or
    empty) — the split gbem_pcg_extract_cmatrix_dev uses."""
    if world < 1:
        raise ValueError("world must be >= 1")
    m = -(-n // world) if n else 0
    return [(min(r * m, n), min((r + 1) * m, n)) for r in range(world)]


class _DevView:
    """Zero-copy torch view of `count` doubles at a device address."""

    def __init__(self, addr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "data": (addr, False),
                                         "version": 3, "strides": None, "stream": None}


class HostCollectives:
    """gbem_collectives over a torch.distributed group whose backend works on
    host tensors (gloo): device buffers are staged through host memory.  With
    ``device=False`` the pointers are host memory (CPU-only tests of the
    callbacks themselves)."""

    def __init__(self, group=None, device: bool = True):
        import torch.distributed as dist
        self.dist, self.group, self.device = dist, group, device
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self._ag = N.AllGatherFn(self._all_gather)
        self._ar = N.AllReduceFn(self._all_reduce)
        self.struct = N.GbemCollectives(None, self._ag, self._ar)
        self.calls = {"all_gather": 0, "all_reduce_sum": 0}

    def _view(self, addr: int, count: int, stream):
        import torch
        if not self.device:
            buf = (C.c_double * count).from_address(addr)
            return torch.from_numpy(np.frombuffer(buf, dtype=np.float64, count=count))
        t = torch.as_tensor(_DevView(addr, count), device="cuda")
        return t

    def _sync(self, stream):
        if self.device:
            import torch
            torch.cuda.synchronize()  # the context's stream (any handle, incl. the legacy default) is on this device

    def _all_gather(self, user, send, recv, count, stream):
        try:
            self._sync(stream)
            s = self._view(send, count, stream).cpu().clone()
            parts = [s.new_empty(count) for _ in range(self.world)]
            self.dist.all_gather(parts, s, group=self.group)
            out = self._view(recv, count * self.world, stream)
            import torch
            out.copy_(torch.cat(parts))
            if self.device:
                torch.cuda.synchronize()
            self.calls["all_gather"] += 1
            return 0
        except Exception:  # noqa: BLE001 — reported to the library as a failed collective
            import traceback
            traceback.print_exc()
            return 1

    def _all_reduce(self, user, buf, count, stream):
        try:
            self._sync(stream)
            v = self._view(buf, count, stream)
            h = v.cpu().clone()
            self.dist.all_reduce(h, group=self.group)
            v.copy_(h)
            if self.device:
                import torch
                torch.cuda.synchronize()
            self.calls["all_reduce_sum"] += 1
            return 0
        except Exception:  # noqa: BLE001
            import traceback
            traceback.print_exc()
            return 1


def attach(ctx, group=None, collectives: str = "auto"):
    """Give ``ctx`` the ranks of ``group`` (default: the world).  collectives:
    "nccl" (the context owns an NCCL communicator), "host" (HostCollectives over
    the group), or "auto" (NCCL iff the group's backend is NCCL).  Returns the
    object that must outlive the context's collective calls (or None)."""
    import torch.distributed as dist
    ctx._coll_keep = None
    if not (dist.is_available() and dist.is_initialized()):
        ctx.check(ctx.lib.gbem_ctx_set_collectives(ctx.h, 1, 0, None))
        return None
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if world == 1:
        ctx.check(ctx.lib.gbem_ctx_set_collectives(ctx.h, 1, 0, None))
        return None
    if collectives == "auto":
        collectives = "nccl" if dist.get_backend(group) == "nccl" else "host"
    if collectives == "nccl":
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            ctx.check(ctx.lib.gbem_nccl_unique_id(C.cast(uid, C.c_void_p)))
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0, group=group)
        uid = (C.c_uint8 * 128).from_buffer_copy(box[0])
        ctx.check(ctx.lib.gbem_ctx_init_nccl(ctx.h, world, rank, C.cast(uid, C.c_void_p)))
        return None
    hc = HostCollectives(group)
    ctx.check(ctx.lib.gbem_ctx_set_collectives(ctx.h, world, rank, C.byref(hc.struct)))
    ctx._coll_keep = hc  # the callbacks live as long as the context uses them
    return hc


def sharded_cmatrix(ctx, P, net_of_panel: np.ndarray, K: int, eps_r: float, cfg=None, group=None,
                    tol: float = 1e-10, max_iter: int = 1000, jacobi_blocks: int = 1, collectives: str = "auto",
                    attach_ranks: bool = True):
    """C-matrix on row-block shards through the host-buffer entry point
    ``gbem_pcg_extract_cmatrix`` (panel and net upload, C / resid / outer
    download inside the call); every rank of ``group`` calls it with the same
    panels (``_native.PanelArrays``).  Returns (C (K, K), resid (K,), outer (K,),
    GbemPcgStats, GbemAssemblyStats); identical on every rank.
    ``attach_ranks=False`` reuses the ranks / collectives attached earlier."""
    if attach_ranks:
        attach(ctx, group, collectives)
    try:
        import torch
        if torch.cuda.is_available():
            ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    except ImportError:
        pass
    net = np.ascontiguousarray(net_of_panel, dtype=np.int32)
    Cm = np.zeros((K, K))
    res = np.zeros(K)
    outer = np.zeros(K)
    opt = N.GbemPcgOptions(tol, max_iter, jacobi_blocks)
    pst, ast = N.GbemPcgStats(), N.GbemAssemblyStats()
    sp = P.struct()
    rc = ctx.lib.gbem_pcg_extract_cmatrix(ctx.h, C.byref(sp), P.n, N.ptr(net), K, eps_r, C.byref(cfg or ctx.quad()),
                                          C.byref(opt), N.ptr(Cm), N.ptr(res), N.ptr(outer), C.byref(ast),
                                          C.byref(pst))
    ctx.check(rc)
    return Cm, res, outer, pst, ast
