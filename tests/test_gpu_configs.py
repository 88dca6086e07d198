"""Full-size BASELINE configs 3-5 on the GPU: complete rows of the assembled
matrix (gbem_assemble_rows_full_dev, the sharded path) at sampled row indices,
checked entry by entry against the CPU oracle with the two-sided gate of
test_gpu_pairs.py.  The CPU oracle cannot assemble these
matrices whole (config 5 is 2e10 entries), so the rows are sampled: every near
pair (gap/diameter < 1.5) of the sampled rows plus a seeded sample of far
pairs, with the per-entry scaling U / (|I_i| |I_j|) of assembly.hpp:96-99."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle_lib as O
import paper_2203_11733_b200 as g
from paper_2203_11733_b200 import _native as N
from paper_2203_11733_b200.shard import panels_to_device
from test_gpu_pairs import _gate

pytestmark = pytest.mark.gpu


def _rows_of(ctx, ps, rows):
    """Full row r of A for each sampled r (one full-row assembly launch each)."""
    n = len(ps)
    pd = panels_to_device(ps, torch.device("cuda", 0))
    dp = C.POINTER(C.c_double)
    panels = N.GbemPanels(C.cast(C.c_void_p(pd["axis"].data_ptr()), C.POINTER(C.c_uint8)),
                          *[C.cast(C.c_void_p(pd[k].data_ptr()), dp) for k in ("level", "a0", "a1", "b0", "b1")])
    cfg = ctx.quad()
    ld = ((n + 7) // 8) * 8
    buf = torch.zeros((1, ld), dtype=torch.float64, device="cuda")
    out = {}
    ctx.set_stream(0)
    for r in rows:
        ctx.check(ctx.lib.gbem_assemble_rows_full_dev(ctx.h, C.byref(panels), n, r, r + 1, C.byref(cfg),
                                                      C.c_void_p(buf.data_ptr()), ld, None))
        out[r] = buf[0, :n].cpu().numpy().copy()
    return out


def _gap_ratio_row(P, r):
    """rectDistance / max diameter (geometry.hpp:73,79-87) of panel r against all panels."""
    def ext(M):
        lo = np.empty((len(M), 3)); hi = np.empty((len(M), 3))
        ax = M[:, 0].astype(int)
        for k in range(3):
            i0 = np.where(ax == 0, 1, 0); i1 = np.where(ax == 2, 1, 2)
            lo[:, k] = np.where(ax == k, M[:, 1], np.where(i0 == k, M[:, 2], M[:, 4]))
            hi[:, k] = np.where(ax == k, M[:, 1], np.where(i0 == k, M[:, 3], M[:, 5]))
        return lo, hi
    lo, hi = ext(P)
    d = np.maximum(0.0, np.maximum(lo - hi[r], lo[r] - hi))
    gap = np.sqrt((d * d).sum(1))
    diam = np.hypot(P[:, 3] - P[:, 2], P[:, 5] - P[:, 4])
    return gap / np.maximum(diam, diam[r])


@pytest.mark.parametrize("config,nrows,nfar", [(3, 3, 300), (4, 2, 300), (5, 4, 300)])
def test_config_rows_match_oracle(ctx, config, nrows, nfar):
    m = g.config_model(config, seed=1)
    ps = m.partition(1)
    P = ps.matrix()
    n = len(P)
    rng = np.random.default_rng(config)
    rows = sorted(rng.choice(n, size=nrows, replace=False).tolist())
    got = _rows_of(ctx, ps, rows)
    area = (P[:, 3] - P[:, 2]) * (P[:, 5] - P[:, 4])
    for r in rows:
        gr = _gap_ratio_row(P, r)
        near = np.flatnonzero(gr < 1.5)
        far = np.flatnonzero(gr >= 1.5)
        cols = np.concatenate([near[:400], rng.choice(far, size=min(nfar, len(far)), replace=False)])
        A = np.repeat(P[r:r + 1], len(cols), axis=0)
        B = P[cols]
        ref, conv, _ = O.u_pairs("orc", A, B, nthreads=16)
        gg = gr[cols]
        truth = ref.copy()
        fm = gg >= 1.5
        if fm.any():
            truth[fm] = O.truth_pairs(A[fm], B[fm])
        gpu = got[r][cols] * area[r] * area[cols]
        touching = gg == 0
        bad, e1 = _gate(gpu, ref, truth, gg, touching)
        assert not bad.any(), (config, r, int(bad.sum()), float(e1.max()), cols[np.argmax(e1)])
        assert np.all(np.isfinite(got[r]))
