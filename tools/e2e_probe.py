"""Per-call wall time of the host-buffer extraction (gbem_extract_cmatrix) on
the bench workload, to look at e2e jitter (diagnostic)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
from paper_2203_11733_b200 import _native as N

m, ps, net, K, eps = bench.workload(2, 1)
ctx = N.Context(0)
P = ps.arrays()
ts = []
for k in range(30):
    t0 = time.perf_counter()
    ctx.extract_cmatrix(P, net, K, eps, stats=False)
    ts.append(1e3 * (time.perf_counter() - t0))
print("per-call ms:", " ".join(f"{t:.1f}" for t in ts))
ast, sst = N.GbemAssemblyStats(), N.GbemSolveStats()
Cm, res, ast, sst = ctx.extract_cmatrix(P, net, K, eps, stats=True)
print("stats call:", ast.ms_total, sst.ms_factor, sst.ms_solve)
