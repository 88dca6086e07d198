"""Full-size runs of BASELINE configs 1-5 on one B200 (not the bench: minutes).

  configs 1-4: C-matrix extraction through gbem_extract_cmatrix_dev (assembly +
               DMMA Cholesky + K solves + charges), device-timed phases,
               C-matrix sanity (reciprocity, signs, residuals);
  config 4:    additionally the row-block block-Jacobi PCG (gbem_pcg_extract_cmatrix_dev) with 8
               Jacobi blocks (the 8-rank preconditioner on one GPU) against the
               direct C-matrix;
  config 5:    assembly only, streamed through 16 full-row blocks.
Prints one JSON object per config.  python tools/run_configs.py [ids...]
"""
import ctypes as C
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2203_11733_b200 as g
from paper_2203_11733_b200 import _native as N
from paper_2203_11733_b200.pcg import sharded_cmatrix
from paper_2203_11733_b200.shard import panels_to_device


def workload(config):
    m = g.config_model(config, seed=1)
    ps = m.partition(1)
    ids = m.net_ids
    col = {nid: k for k, nid in enumerate(ids)}
    net = np.array([col.get(int(v), -1) if k == 0 else -1 for v, k in zip(ps.net, ps.kind)], dtype=np.int32)
    return m, ps, net, len(ids), m.info()["eps_r"]


def direct(config):
    m, ps, net, K, eps = workload(config)
    n = len(ps)
    ctx = N.Context(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    pd = panels_to_device(ps, torch.device("cuda", 0))
    dp = C.POINTER(C.c_double)
    panels = N.GbemPanels(C.cast(C.c_void_p(pd["axis"].data_ptr()), C.POINTER(C.c_uint8)),
                          *[C.cast(C.c_void_p(pd[k].data_ptr()), dp) for k in ("level", "a0", "a1", "b0", "b1")])
    d_net = torch.from_numpy(net).cuda()
    d_C = torch.zeros(K * K, dtype=torch.float64, device="cuda")
    d_res = torch.zeros(K, dtype=torch.float64, device="cuda")
    ast, sst = N.GbemAssemblyStats(), N.GbemSolveStats()
    cfg = ctx.quad()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # twice in one context: the first extraction also allocates the context's
    # buffers (matrix, pair queue) and loads modules; the second is the steady state
    times = []
    for _ in range(2):
        t0 = time.perf_counter()
        e0.record()
        ctx.check(ctx.lib.gbem_extract_cmatrix_dev(ctx.h, C.byref(panels), n, C.c_void_p(d_net.data_ptr()), K,
                                                   eps, C.byref(cfg), C.c_void_p(d_C.data_ptr()),
                                                   C.c_void_p(d_res.data_ptr()), C.byref(ast), C.byref(sst)))
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = times[-1]
    Cm = d_C.cpu().numpy().reshape(K, K)
    res = d_res.cpu().numpy()
    entries = n * (n + 1) // 2
    recip = float(np.max(np.abs(Cm - Cm.T)) / np.max(np.abs(np.diag(Cm))))
    off = Cm[~np.eye(K, dtype=bool)]
    out = dict(config=config, panels=n, nets=K, entries=entries, matrix_gb=n * n * 8 / 1e9,
               extraction_ms=ms, first_extraction_ms=times[0], wall_s=time.perf_counter() - t0, entries_per_s=entries / (ast.ms_total * 1e-3),
               assembly=ast.as_dict(), solve=sst.as_dict(),
               cholesky_tflops=(n ** 3 / 3) / (sst.ms_factor * 1e-3) / 1e12,
               max_residual=float(res.max()), reciprocity_defect=recip,
               diag_positive=bool(np.all(np.diag(Cm) > 0)), offdiag_negative=bool(np.all(off < 0)),
               c_diag_first=[float(x) for x in np.diag(Cm)[:4]])
    ctx.close()
    del pd, d_net, d_C, d_res
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out, Cm


def pcg_vs_direct(config, Cd, blocks=8, tol=1e-10):
    m, ps, net, K, eps = workload(config)
    ctx = N.Context(0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Cp, res, _, st, ast = sharded_cmatrix(ctx, ps.arrays(), net, K, eps, tol=tol, max_iter=2000, jacobi_blocks=blocks)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    rel = float(np.max(np.abs(Cp - Cd)) / np.max(np.abs(Cd)))
    ctx.close()
    torch.cuda.empty_cache()
    return dict(config=config, jacobi_blocks=blocks, tol=tol, wall_s=wall, cmatrix_max_rel_diff_vs_direct=rel,
                matvec_tflops=st.matvec_flops / (st.ms_matvec * 1e-3) / 1e12, **st.as_dict())


def stream_assembly(config=5, chunks=16):
    from paper_2203_11733_b200.shard import ShardedAssembler
    ps = g.config_model(config, seed=1).partition(1)
    n = len(ps)
    ctx = N.Context(0)
    ctx.set_stream(0)
    pd = panels_to_device(ps, torch.device("cuda", 0))
    tot = 0
    chk = torch.zeros((), dtype=torch.float64, device="cuda")
    stats = dict(far=0, cop=0, par=0, orth=0, nonconv=0, ms_far=0.0, ms_near=0.0, ms_cls=0.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for c in range(chunks):
        sh = ShardedAssembler(ctx, pd, n, c, chunks)
        blk = sh.assemble(with_stats=True)
        chk += blk.sum()
        st = sh.stats
        tot += st.pairs_total
        for k, f in (("far", "pairs_far"), ("cop", "pairs_coplanar"), ("par", "pairs_parallel"),
                     ("orth", "pairs_orthogonal"), ("nonconv", "not_converged"), ("ms_far", "ms_far"),
                     ("ms_near", "ms_near"), ("ms_cls", "ms_classify")):
            stats[k] += getattr(st, f)
        del sh, blk
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ctx.close()
    return dict(config=config, panels=n, entries=tot, ms=ms, entries_per_s=tot / (ms * 1e-3),
                checksum=float(chk), **stats)


if __name__ == "__main__":
    ids = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5]
    for c in ids:
        if c == 5:
            print(json.dumps(stream_assembly()), flush=True)
            continue
        out, Cd = direct(c)
        print(json.dumps(out), flush=True)
        if c == 4:
            print(json.dumps(pcg_vs_direct(c, Cd)), flush=True)
